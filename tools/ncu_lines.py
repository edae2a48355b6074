#!/usr/bin/env python
"""Per-source-line warp-stall / instruction attribution of one kernel in an
ncu report (SASS page) using the line table of the built library.

  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED_SUBSTR [LIB.so] [TOP]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, fn = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "paper_2003_05361_b200",
                                                             "libras_b200.so")
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
    addr2line = {}
    for cub in os.listdir(tmp):
        sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
        lines = sass.splitlines()
        start = None
        for i, l in enumerate(lines):
            if ".section" in l and ".text." in l and fn in l:
                start = i
                break
        if start is None:
            continue
        cur = None
        for l in lines[start + 1:]:
            if l.strip().startswith(".section") and ".text." in l:
                break
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
            if m:
                addr2line[int(m.group(1), 16)] = cur
        break
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    base = min(int(r[0], 16) for r in data)
    agg = {}
    for r in data:
        k = addr2line.get(int(r[0], 16) - base) or ("?", 0)
        a = agg.setdefault(k, [0.0, 0.0])
        a[0] += float(r[iS] or 0)
        a[1] += float(r[iE] or 0)
    tot = sum(v[0] for v in agg.values())
    srcs = {}
    for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        text = ""
        for root, _, files in os.walk(os.path.join(os.path.dirname(__file__), "..", "paper_2003_05361_b200")):
            if f in files:
                p = os.path.join(root, f)
                if p not in srcs:
                    srcs[p] = open(p).read().splitlines()
                text = srcs[p][ln - 1].strip() if 0 < ln <= len(srcs[p]) else ""
        print(f"{100 * v[0] / tot:5.1f}%  {int(v[1]):>11d}  {f}:{ln}  {text[:90]}")


if __name__ == "__main__":
    main()
