import sys
import numpy as np
for f in sys.argv[1:]:
    t = np.fromfile(f, dtype=np.uint64)[:160 * 64 * 4].reshape(160, 64, 4).astype(np.int64)[:148, :20]
    t = t - t[:, 0, 0].min()
    A = (t[:, :, 1] - t[:, :, 0]).mean() / 1e3
    B = (t[:, :, 3] - t[:, :, 2]).mean() / 1e3
    rel = np.mean([(t[:, i, 2].min() - t[:, i, 1].max()) / 1e3 for i in range(1, 20)])
    spread = np.mean([(t[:, i, 1].max() - t[:, i, 1].min()) / 1e3 for i in range(1, 20)])
    it = np.mean([(t[:, i + 1, 0].min() - t[:, i, 0].min()) / 1e3 for i in range(1, 19)])
    print(f"{f}: iter {it:.2f} us | passA {A:.2f} | passB {B:.2f} | arrival spread {spread:.2f} | last arrival->first release {rel:.2f}")

# reduction internals (second block of the file, if present): per reduction k
for f in sys.argv[1:]:
    a = np.fromfile(f, dtype=np.uint64)
    if a.size < 2 * 160 * 64 * 4:
        continue
    r = a[160 * 64 * 4:].reshape(160, 64, 4).astype(np.int64)[:148, 20:40]  # reductions of a later subdomain
    ks = range(r.shape[1])
    arrive_last = np.array([r[:, k, 0].max() for k in ks])
    stored_last = np.array([r[:, k, 1][np.argmax(r[:, k, 0])] for k in ks])
    polled_first = np.array([r[:, k, 2].min() for k in ks])
    polled_med = np.array([np.median(r[:, k, 2]) for k in ks])
    rel_last = np.array([r[:, k, 3].max() for k in ks])
    print("last CTA: arrive->stored %.2f us | stored->first poll done %.2f | ->median poll done %.2f | ->last release %.2f"
          % (np.mean(stored_last - arrive_last) / 1e3, np.mean(polled_first - stored_last) / 1e3,
             np.mean(polled_med - stored_last) / 1e3, np.mean(rel_last - stored_last) / 1e3))
