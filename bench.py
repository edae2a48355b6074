#!/usr/bin/env python
"""Benchmark of the B200-native RAS hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1] = C2 at N=1; C3-style weak scaling at N>1):
2D 5-point Laplacian, 1024x1024 owned unknowns per subdomain, 16 subdomains per
GPU (4x4 tiles at N=1: 4096^2 = 16.8M unknowns), overlap 8, Jacobi-PCG m=20,
synchronous RAS.  One "step" = one RAS sweep over the whole problem (restrict,
residual, local solves, restricted prolongation, exchange, global check).

value     = RAS iterations/s = sync sweeps / s (max over ranks); the aggregate
            subdomain updates/s (subdomains x sweeps/s) is the extra key `subdomain_updates_per_s`
e2e       = the same through the public API with pinned HOST x0 / x_out (each rank its owned values), copies inside
roofline  = dominant kernel: algorithmic bytes / CUDA-event duration vs measured HBM copy peak
spmv_gbs  = the residual SpMV (k_residual, a1+a2): algorithmic bytes / event time
tts       = time-to-solution to rel. residual 1e-8 (P474-480) on C1 and the 256^2 / 512^2
            analogues of C2 (sync and async), with the oracle's full TTS beside it where it
            finishes in seconds (C1, 256^2)
cpu_baseline = the oracle (rank 0, N=1): K=3 full sync sweeps of this workload, plus the oracle
            TTS above and an extrapolated C2 TTS (labelled)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode sync|async]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ras_inputs as ri  # noqa: E402

SUB = 1024          # owned unknowns per subdomain side
PER_GPU = (4, 4)    # subdomain tiles per GPU
GAMMA = 8
M_INNER = 20
TILES = {1: (4, 4), 2: (4, 8), 4: (8, 8), 8: (8, 16)}


def workload(N):
    px, py = TILES.get(N, (4, 4 * N))
    return px, py, px * SUB, py * SUB


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="sync", choices=["sync", "async"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the small-config time-to-solution runs")
    ap.add_argument("--config", default="c2", choices=["c2", "c5"],
                    help="c2: C2 at N=1 / C3-style weak scaling at N>1 (default); c5: C5-shaped weak scaling "
                         "(8 balanced irregular cells of ~1.56 M unknowns per GPU; 10^8 at N=8)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--tts", action="store_true", help="also run to rel. residual 1e-8 (long)")
    ap.add_argument("--scale", type=int, default=SUB, help="owned side per subdomain (debug)")
    ap.add_argument("--plain", action="store_true", help="force plain FP64/int32 SELL (default: SELL-Z when it applies)")
    ap.add_argument("--fuse-p", action="store_true", help="fuse the PCG p update into the next SpMV")
    ap.add_argument("--path", default="auto", choices=["auto", "tiled", "block", "resident"],
                    help="local-PCG execution path (ras_pcg_path)")
    ap.add_argument("--robin", type=float, default=0.0, help="ORAS transmission parameter (0 = RAS, the C2 config)")
    ap.add_argument("--overlap", type=int, default=GAMMA, help="overlap gamma (8 = the C2 config; C3 sweeps 1/2/4/8)")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)
# ----------------------------------------------------------------------------
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    def __init__(self, devices):
        self.devices = devices
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", ",".join(str(d) for d in self.devices)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~1 s before its first sample: wait for it so the
            # samples cover the timed region that follows
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.05)
        except OSError:
            self.proc = None
        self.window = [None, None]
        return self

    def mark(self, i):
        self.window[i] = time.time()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(1)

    def summary(self):
        sm, mx, reasons = [], [], set()
        w0, w1 = self.window
        for ts, ln in self.lines:
            if w0 is not None and w1 is not None and not (w0 - 0.06 <= ts <= w1 + 0.06):
                continue  # keep samples taken during the timed region
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(REASONS, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_onchip(kernel):
    """On-chip counters of `kernel` from the committed ncu summary (profiles/ncu_onchip.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_onchip.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def build_rank_problem(N, rank, scale=SUB, config="c2"):
    """Row window of the global Laplacian + RHS + owner array for one rank.
    config "c5": BASELINE configs[4] shape per GPU -- 8 balanced irregular cells of
    ~1.56 M unknowns per GPU (Voronoi + Lloyd + power-diagram balancing, the graph-
    partitioner stand-in), N x 12.5 M unknowns in total (10^8 at N = 8)."""
    from paper_2003_05361_b200 import partition_regular

    if config == "c5":
        import numpy as np_

        side = int(round((12.5e6 * N) ** 0.5))
        P = 8 * N
        owner = ri.voronoi_partition(side, side, P, seed=1, lloyd=8, balance=60)
        s2r = (np_.arange(P) * N) // P
        rows = np_.nonzero(s2r[owner] == rank)[0]
        r0 = max(0, int(rows.min()) - (GAMMA + 1) * side)
        r1 = min(side * side, int(rows.max()) + 1 + (GAMMA + 1) * side)
        A = ri.laplace_2d_rows(side, side, r0, r1)
        b = ri.rhs_rows(side * side, r0, r1, 0)
        return dict(nx=side, ny=side, n=side * side, P=P, px=0, py=0, owner=owner, A=A, b=b)

    px, py = TILES.get(N, (4, 4 * N))
    nx, ny = px * scale, py * scale
    n = nx * ny
    owner = partition_regular(nx, ny, 1, px, py, 1)
    P = px * py
    s0, s1 = (rank * P) // N, ((rank + 1) * P) // N  # contiguous subdomain ids (default sub_to_rank)
    ty0, ty1 = s0 // px, (s1 - 1) // px + 1            # tile rows of this rank
    r0 = max(0, ty0 * scale - (GAMMA + 1))
    r1 = min(ny, ty1 * scale + (GAMMA + 1))
    A = ri.laplace_2d_rows(nx, ny, r0 * nx, r1 * nx)
    b = ri.rhs_rows(n, r0 * nx, r1 * nx, 0)
    return dict(nx=nx, ny=ny, n=n, P=P, px=px, py=py, owner=owner, A=A, b=b)


# ----------------------------------------------------------------------------
# reference arm and cpu baseline: the oracle, as it stands, on host cores
# ----------------------------------------------------------------------------
def oracle_setup(nx, ny, px, py, gamma, kind, m):
    import oracle as O

    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    owner = O.partition_regular(nx, ny, 1, px, py, 1)
    subs = O.setup(A, b, owner, gamma)
    for s_ in subs:
        O.make_local_solver(s_, kind, m)
    return A, b, subs


def oracle_sweeps(nx, ny, px, py, K=3):
    """K full synchronous oracle sweeps of the workload (Alg. 1 loop: global check,
    every subdomain's residual + Jacobi-PCG(m) + restricted prolongation), one BLAS
    thread; setup untimed (P229-231).  Returns (sweeps/s, details)."""
    from threadpoolctl import threadpool_limits

    import oracle as O

    with threadpool_limits(1):
        t0 = time.perf_counter()
        A, b, subs = oracle_setup(nx, ny, px, py, GAMMA, "jacobi", M_INNER)
        t1 = time.perf_counter()
        O.ras_sync(A, b, subs, 1e-300, K)
        t2 = time.perf_counter()
    return K / (t2 - t1), {"sweeps": K, "solve_s": t2 - t1, "setup_s": t1 - t0}


def oracle_tts(nx, ny, px, py, gamma, kind, m, tol=1e-8):
    """Full oracle time-to-solution (sync, setup untimed), one BLAS thread."""
    from threadpoolctl import threadpool_limits

    import oracle as O

    with threadpool_limits(1):
        A, b, subs = oracle_setup(nx, ny, px, py, gamma, kind, m)
        t0 = time.perf_counter()
        r = O.ras_sync(A, b, subs, tol, 200000)
        t1 = time.perf_counter()
    return {"time_s": t1 - t0, "sweeps": r.sweeps, "cores": 1}


# time-to-solution configurations: C1 and analogues of C2 at smaller N
TTS_CFGS = [
    # name, N, tiles per side, overlap, local solver, m, oracle TTS in the default run
    ("C1", 64, 2, 2, "exact", 0, True),
    ("C2@256", 256, 4, 8, "jacobi", 20, True),
    ("C2@512", 512, 4, 8, "jacobi", 20, False),  # oracle: 1914 sweeps, ~175 s on one core
]


def oracle_sample(nx, ny, P, px, sample_subs, sweeps_per_sub, budget_s=25.0):
    """Time the oracle's per-subdomain work of a sync sweep (local residual +
    Jacobi-PCG(m) + restricted prolongation) on `sample_subs` subdomains of the
    bench workload, plus the oracle's global residual check; return
    (subdomain updates per second, details)."""
    from threadpoolctl import threadpool_limits

    import oracle as O

    A = ri.laplace_2d(nx, ny)
    b = ri.rhs(nx * ny, 0)
    owner = O.partition_regular(nx, ny, 1, px, P // px, 1)
    As = O.as_scipy(A)
    x = np.zeros(nx * ny)
    times = []
    with threadpool_limits(1):
        for p in sample_subs:
            om, ow, gh = O.overlap_sets(As, owner, p, GAMMA)
            rows = As[om]
            sub = O.Subdomain(p, om, ow, gh, rows[:, om].tocsr(), rows[:, gh].tocsr(), b[om].copy())
            O.make_local_solver(sub, "jacobi", M_INNER)
            for _ in range(sweeps_per_sub):
                t0 = time.perf_counter()
                rt = O.local_residual(sub, x)
                d = sub.solver(rt)
                og = sub.owned_global
                x[og] = x[og] + d[sub.owned]
                times.append(time.perf_counter() - t0)
            if sum(times) > budget_s:
                break
        t0 = time.perf_counter()
        r = b - As @ x
        _ = float(np.linalg.norm(r)) / float(np.linalg.norm(b))
        t_res = time.perf_counter() - t0
    t_sub = statistics.mean(times)
    sweep_s = P * t_sub + t_res
    return P / sweep_s, {"t_sub_update_s": t_sub, "t_global_residual_s": t_res, "sweep_s": sweep_s,
                         "samples": len(times)}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    N = args.gpus
    px, py, nx, ny = workload(N) if args.scale == SUB else (4, 4, 4 * args.scale, 4 * args.scale)
    P = px * py
    steps = max(1, args.steps)
    warm = max(0, args.warmup)
    # one reference "step" = one sampled subdomain update (+1/P of the global residual);
    # a full oracle sweep of C2 (16 updates + the global check) takes ~5 s on one core
    t0 = time.perf_counter()
    upd, det = oracle_sample(nx, ny, P, px, [5, 6], max(1, (steps + warm + 1) // 2), budget_s=120.0)
    wall = time.perf_counter() - t0
    val = 1.0 / det["sweep_s"]  # sweeps/s
    line = {
        "impl": "reference", "metric": METRIC, "value": val,
        "unit": "sweeps/s", "n_gpus": N, "steps": steps, "warmup": warm,
        "ms_per_step": det["sweep_s"] * 1000.0 / P, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(N, nx, ny, P, "sync"),
        "subdomain_updates_per_s": upd,
        "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle (NumPy/SciPy, 1 thread) local residual + Jacobi-PCG(m={M_INNER}) + prolong "
                                   f"on subdomains 5,6 of the workload, {det['samples']} updates (one per step), plus one "
                                   f"global residual; sweep time = P*t_update + t_residual = {det['sweep_s']:.2f} s",
                         "host_cores_available": os.cpu_count()},
        "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "RAS iterations/s (sync sweeps/s); time-to-solution to 1e-8 in `tts`; SpMV GB/s in `spmv_gbs`"


def config_dict(N, nx, ny, P, mode, config="c2"):
    # identical in both arms (the driver compares them); the working set of the
    # sweep (r, p, d, b, x, matrix ~ 12 B/row) is >= 1.3 GB per GPU at C2 >> 126 MB L2
    ws = 8.0 * nx * ny * 10
    if config == "c5":
        name = (f"C5-shaped: 2D 5-pt Laplacian {nx}x{ny} ({nx * ny / 1e6:.1f}M unknowns), {P} balanced irregular "
                f"(graph-partition stand-in) subdomains ({P // N}/GPU), overlap {GAMMA}, Jacobi-PCG m={M_INNER}, {mode} RAS")
    else:
        name = (f"{'C2' if N == 1 else 'C3-weak'}: 2D 5-pt Laplacian {nx}x{ny} ({nx * ny / 1e6:.1f}M unknowns), "
                f"{P} subdomains of {SUB}^2 ({P // N}/GPU), overlap {GAMMA}, Jacobi-PCG m={M_INNER}, {mode} RAS")
    return {"workload": name,
            "grid": [nx, ny], "subdomains": P, "subdomains_per_gpu": P // N, "overlap": GAMMA,
            "inner_iters": M_INNER, "mode": mode, "precision": "fp64",
            "parallelism": f"domain decomposition, {P // N} subdomains per GPU x {N} GPU",
            "l2": f"inputs > L2: working set ~{ws / N / 1e9:.1f} GB per GPU >> 126 MB L2, no flush needed"}


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------
def main():
    global GAMMA
    args = parse()
    GAMMA = args.overlap
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2003_05361_b200 as R

    rank, world, local = dist_env()
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:
        obj = [R.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t_setup0 = time.perf_counter()
    prob = build_rank_problem(N, rank, args.scale, args.config)
    opts = R.options("jacobi", M_INNER, plain=args.plain, fuse_p=args.fuse_p, path=args.path, robin=args.robin)
    solver = R.Solver(prob["A"], prob["b"], prob["owner"], GAMMA, opts,
                      comm={"rank": rank, "world": world, "device": local, "nccl_id": nccl_id,
                            "stream": stream.cuda_stream})
    del prob["A"]
    setup_s = time.perf_counter() - t_setup0
    info = solver.plan().info()
    P, nx, ny, n = prob["P"], prob["nx"], prob["ny"], prob["n"]
    mode = args.mode

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # warm-up (untimed)
    if args.warmup > 0:
        solver.solve_device(1e-300, args.warmup, mode)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler([local] if world == 1 else list(range(world))) as clk:
        barrier()
        clk.mark(0)
        e0.record(stream)
        st = solver.solve_device(1e-300, args.steps, mode)
        e1.record(stream)
        barrier()
        clk.mark(1)
    ms_local = e0.elapsed_time(e1)
    stats = solver.stats()
    # per-kernel breakdown: the same K sweeps again with every launch bracketed by
    # CUDA events on the library stream (events between launches disable the
    # programmatic-dependent-launch overlap, so this pass is not the value pass)
    solver.kernel_timing(True)
    barrier()
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    # per-kernel event timing runs on the library stream, i.e. the sync schedule;
    # the async mode launches the same kernels per subdomain stream
    solver.solve_device(1e-300, args.steps, "sync")
    k1.record(stream)
    barrier()
    ms_kpass = k0.elapsed_time(k1)
    ktimes = solver.kernel_times()
    solver.kernel_timing(False)
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    sweeps = stats["sweeps"] if mode == "sync" else stats["updates_max"]
    value = args.steps / (ms / 1e3)  # RAS iterations (sync sweeps) / s, Q27
    updates_per_s = P * value      # aggregate subdomain updates / s (all ranks)

    # roofline: dominant kernel by event time.  A whole-solve kernel (RESIDENT /
    # BLOCK path: every PCG iteration of every subdomain in one launch) is rated
    # on the bytes the same iterations move when streamed by the tiled kernels
    # (DESIGN.md §5 model x inner iterations) -- its actual HBM traffic is only
    # the compulsory once-per-sweep part, reported as "compulsory_bytes".
    tot_ms = sum(v[1] for v in ktimes.values())
    per_it = sum(ktimes[k][2] for k in ("k_spmv_dot", "k_update_dot", "k_pupdate") if k in ktimes)
    kern = {}
    for name, (cnt, kms, bpl) in ktimes.items():
        if cnt == 0:
            continue
        avg_ms = kms / cnt
        rec = {"launches": cnt, "avg_us": avg_ms * 1e3, "share": kms / tot_ms if tot_ms else None}
        if name in ("k_resident_pcg", "k_resident2", "k_small_pcg"):
            rec["compulsory_bytes"] = bpl
            bpl = per_it * M_INNER + ktimes["k_prolong"][2]
        rec["bytes_per_launch"] = bpl
        rec["gbs"] = (bpl / (avg_ms / 1e3) / 1e9) if bpl and avg_ms > 0 else None
        kern[name] = rec
    dom = max((k for k in kern if kern[k]["bytes_per_launch"]), key=lambda k: kern[k]["share"] or 0)
    peak, peak_src = measured_peaks()
    tr = ncu_traffic(dom)
    if dom in ("k_resident2", "k_resident_pcg"):
        # the whole local solve runs on chip: its HBM traffic is only the compulsory
        # once-per-sweep part, so the bound is ON-CHIP.  Model ("RESIDENT
        # roofline"): algorithmic shared-memory bytes of one PCG iteration of the
        # row-pattern SpMV + update = 5 p reads (40 B) + pattern id (1 B) + p read and
        # write in the update (16 B) = 57 B per Omega-row, x m iterations x rows, against
        # the shared-memory bandwidth 148 SMs x 128 B/clk x 1.965 GHz = 37.2 TB/s (B200
        # unit counts and max clock, B200_PROFILING.md / B300_MICROARCH.md)
        rows = float(stats["rows_local"])
        smem_bytes = 57.0 * rows * M_INNER
        smem_peak = 148 * 128 * 1.965  # GB/s
        avg_s = kern[dom]["avg_us"] * 1e-6
        roof = {"bound": "smem", "kernel": dom, "achieved": smem_bytes / avg_s / 1e9, "peak": smem_peak,
                "unit": "GB/s", "frac": smem_bytes / avg_s / 1e9 / smem_peak, "traffic": tr,
                "peak_source": "derived: 148 SMs x 128 B/clk shared memory x 1.965 GHz (B200 unit counts, max SM clock)",
                "bytes_per_launch": smem_bytes,
                "bytes_model": "on-chip: 57 B of shared memory per Omega-row per PCG iteration (5 p gathers, pattern id, "
                               "p update), x m x rows; r, d live in tensor memory (k_resident2)",
                "hbm": {"compulsory_bytes": kern[dom].get("compulsory_bytes"),
                        "gbs": (kern[dom].get("compulsory_bytes") or 0) / avg_s / 1e9,
                        "frac": (kern[dom].get("compulsory_bytes") or 0) / avg_s / 1e9 / peak,
                        "streamed_model_gbs": kern[dom]["gbs"],
                        "note": "HBM is not this kernel's bound: its DRAM traffic is the compulsory once-per-sweep "
                                "bytes; streamed_model_gbs = the bytes the tiled path would stream for the same "
                                "iterations / launch time (context only)"},
                "ncu": ncu_onchip(dom)}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak, "unit": "GB/s",
                "frac": kern[dom]["gbs"] / peak, "traffic": tr, "peak_source": peak_src,
                "bytes_per_launch": kern[dom]["bytes_per_launch"],
                "bytes_model": "DESIGN.md §5: compulsory bytes of real rows/entries of the streamed (tiled) iteration, "
                               "SELL-Z / int32 SELL indices, FP64 values"}
    pcg_bytes = sum(kern[k]["bytes_per_launch"] * kern[k]["launches"] for k in kern if kern[k]["bytes_per_launch"])
    pcg_ms = sum(ktimes[k][1] for k in kern if kern[k]["bytes_per_launch"])
    # e2e through the public API with pinned HOST buffers: every step copies this
    # rank's owned x0 in and its owned x^{k+1} out (ras_solve_device with host
    # pointers: the distributed form of ras_solve -- no global gather, so the bytes
    # per rank stay constant as N grows); Bi / Bo are summed over the ranks
    e2e = None
    if not args.no_e2e:
        n_own = solver.owned_gids().size
        x0 = torch.zeros(n_own, dtype=torch.float64, pin_memory=True)
        xo = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
        solver.solve_device(1e-300, 1, mode, x0.data_ptr(), xo.data_ptr())  # untimed warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            solver.solve_device(1e-300, 1, mode, x0.data_ptr(), xo.data_ptr())
        barrier()
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = float(te.item())
        e2e = {"value": args.e2e_steps / el, "unit": "sweeps/s", "h2d_bytes_per_step": n * 8,
               "d2h_bytes_per_step": n * 8, "steps": args.e2e_steps,
               "note": "each step = ras_solve_device(x0 = pinned host owned values, max_iters=1, x_out = pinned host "
                       "owned values) on every rank: H2D x0 (+ halo exchange), one sweep + final check, D2H x; bytes "
                       "summed over ranks (= n x 8 each way)"}
    # time-to-solution (P474-480): the bench workload itself only with --tts (C2 needs
    # ~1e5 sweeps, ~7 min); C1 and the 256^2 / 512^2 analogues always at N=1
    tts = {}
    if args.tts:
        barrier()
        t0 = time.perf_counter()
        st = solver.solve_device(1e-8, 200000, mode)
        barrier()
        s2 = solver.stats()
        tts["bench_workload"] = {"time_s": time.perf_counter() - t0, "device_time_s": s2["time_to_solution_s"],
                                 "sweeps": s2["sweeps"], "inner_iters_total": s2["inner_iters_total"],
                                 "final_rel_residual": s2["final_rel_residual"], "converged": bool(s2["converged"])}
    do_small = rank == 0 and N == 1 and not args.no_tts and args.config == "c2"
    if do_small:
        tts.update(gpu_tts_small(R))
    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline and args.config == "c2":
        val, det = oracle_sweeps(nx, ny, prob["px"], prob["py"], K=3)
        o_tts = {}
        if do_small:
            for name, Nn, tiles, g, kind, m, run_oracle in TTS_CFGS:
                if run_oracle:
                    o_tts[name] = oracle_tts(Nn, Nn, tiles, tiles, g, kind, m)
                    tts[name]["oracle"] = o_tts[name]
                    tts[name]["speedup_vs_oracle"] = o_tts[name]["time_s"] / tts[name]["sync"]["time_s"]
        c2_sweeps = committed_c2_sweeps()
        cpu = {"value": val, "unit": "sweeps/s", "cores": 1, "kind": "oracle",
               "sample": f"{det['sweeps']} full synchronous oracle sweeps of this workload (NumPy/SciPy, BLAS limited "
                         f"to 1 thread; {det['solve_s']:.1f} s, setup {det['setup_s']:.1f} s untimed); oracle full "
                         f"time-to-solution on C1 and the 256^2 analogue in tts.*.oracle",
               "host_cores_available": os.cpu_count(),
               "oracle_tts": o_tts,
               "c2_tts_extrapolated_s": (c2_sweeps / val) if c2_sweeps else None,
               "c2_tts_extrapolation": (f"EXTRAPOLATED: {c2_sweeps} sweeps (GPU sync run to 1e-8, "
                                        "profiles/bench_r02_tts_c2.json) / oracle sweeps per s" if c2_sweeps else None)}
    clocks = clk.summary()
    if rank == 0:
        res = kern.get("k_residual")
        line = {
            "metric": METRIC, "value": value, "unit": "sweeps/s",
            "n_gpus": N, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(N, nx, ny, P, mode, args.config),
            "subdomain_updates_per_s": updates_per_s,
            "spmv_gbs": res["gbs"] if res else None,
            "spmv_frac": (res["gbs"] / peak) if res else None,
            "spmv_note": "k_residual (a1+a2: restrict + [A_p | B_p] SpMV + Eq. 2 / owned norms), algorithmic bytes "
                         "(DESIGN.md §5) / CUDA-event launch time",
            "sweeps_done": sweeps,
            "inner_iters_total": stats["inner_iters_total"],
            "pcg_path": ["auto", "tiled", "block", "resident"][stats["pcg_path"]],
            "robin": args.robin,
            "roofline": roof,
            "pcg_path_gbs": pcg_bytes / (pcg_ms / 1e3) / 1e9 if pcg_ms else None,
            "kernels": kern,
            "kernel_pass_ms_per_step": ms_kpass / args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": stats["kernel_launches"],
            "setup_s": setup_s,
            "tts": tts or None,
            "phase_s": {k: stats[k] for k in ("t_residual", "t_local_solve", "t_prolong", "t_exchange", "t_convcheck")},
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def committed_c2_sweeps():
    """GPU sweep count of the committed C2 sync run to 1e-8 (for the labelled extrapolation)."""
    try:
        with open(os.path.join(ROOT, "profiles", "bench_r02_tts_c2.json")) as f:
            d = json.load(f)
        t = d.get("tts") or {}
        t = t.get("bench_workload", t)
        return int(t["sweeps"]) if t.get("converged") else None
    except (OSError, ValueError, KeyError, TypeError):
        return None


def gpu_tts_small(R):
    """Time-to-solution to 1e-8 on C1 and the C2 analogues (sync and async), one GPU."""
    import torch

    out = {}
    for name, Nn, tiles, g, kind, m, _ in TTS_CFGS:
        A = ri.laplace_2d(Nn)
        b = ri.rhs(Nn * Nn, 0)
        owner = R.partition_regular(Nn, Nn, 1, tiles, tiles, 1)
        s = R.Solver(A, b, owner, g, R.options(kind, max(m, 1)))
        rec = {"config": f"{Nn}x{Nn} 2D Laplacian, {tiles}x{tiles} subdomains, overlap {g}, "
                         f"{'exact (PCG to 1e-14)' if kind == 'exact' else f'Jacobi-PCG m={m}'}"}
        for mode in ("sync", "async"):
            s.solve(1e-8, 200000, mode, gather=False)  # warm-up (graphs, first-use buffers)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, _ = s.solve(1e-8, 200000, mode, gather=False)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            t = s.stats()
            rec[mode] = {"time_s": el, "device_tts_s": t["time_to_solution_s"], "sweeps": t["sweeps"],
                         "updates_min": t["updates_min"], "updates_max": t["updates_max"],
                         "inner_iters_total": t["inner_iters_total"], "final_rel_residual": t["final_rel_residual"],
                         "converged": bool(t["converged"]), "verified": bool(t["verified"]),
                         "pcg_path": ["auto", "tiled", "block", "resident"][t["pcg_path"]]}
        s.close()
        out[name] = rec
    return out


if __name__ == "__main__":
    sys.exit(main())
