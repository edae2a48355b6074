"""Thin Python binding over the C ABI (include/ras.h, include/ras_plan.h).

Argument marshalling only: every step of the RAS path runs in libras_b200.so's
CUDA kernels.  PyTorch is used, when present, only for the CUDA stream and the
process group that broadcasts the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _ffi as F
from ._ffi import RasError

__all__ = ["Plan", "Solver", "partition_regular", "options", "RasError", "nccl_unique_id"]


def _check(st, ctx=None):
    if st != F.RAS_OK:
        msg = F.lib().ras_last_error(ctx)
        raise RasError(st, msg.decode() if msg else "")


def _csr_struct(A, n=None):
    """A: object with indptr/indices/data (+ n, row0) or a scipy CSR matrix."""
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int32)
    data = np.ascontiguousarray(A.data, dtype=np.float64)
    nrows = len(indptr) - 1
    gn = int(getattr(A, "n", None) or (n if n is not None else A.shape[1]))
    row0 = int(getattr(A, "row0", 0))
    s = F.RasCsr(gn, row0, nrows, F.ptr(indptr, F.I64), F.ptr(indices, F.I32), F.ptr(data, F.F64))
    return s, (indptr, indices, data)


def _partition_struct(owner, num_subdomains=None, sub_to_rank=None):
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    P = int(num_subdomains if num_subdomains is not None else owner.max() + 1)
    s2r = None if sub_to_rank is None else np.ascontiguousarray(sub_to_rank, dtype=np.int32)
    return F.RasPartition(P, F.ptr(owner, F.I32), F.ptr(s2r, F.I32)), (owner, s2r)


def partition_regular(nx, ny, nz, px, py, pz) -> np.ndarray:
    """ras_partition_regular (P277-286, R23)."""
    out = np.empty(nx * ny * nz, dtype=np.int32)
    _check(F.lib().ras_partition_regular(nx, ny, nz, px, py, pz, F.ptr(out, F.I32)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(F.lib().ras_nccl_unique_id(buf))
    return buf.raw


_SOLVERS = {"jacobi": F.RAS_LS_JACOBI_PCG, "ic0": F.RAS_LS_IC0_PCG, "ilu0": F.RAS_LS_ILU0_PCG,
            "exact": F.RAS_LS_EXACT_PCG, "cholesky": F.RAS_LS_CHOLESKY}
_DETECTORS = {"central": F.RAS_DET_CENTRAL, "decentral": F.RAS_DET_DECENTRAL}


_PATHS = {"auto": F.RAS_PCG_AUTO, "tiled": F.RAS_PCG_TILED, "block": F.RAS_PCG_BLOCK,
          "resident": F.RAS_PCG_RESIDENT}


def options(local_solver="jacobi", inner_iters=20, inner_tol=0.0, detector="decentral", fuse_p=False,
            plain=False, stage=False, tiled=False, path="auto", robin=0.0, **kw) -> F.RasOptions:
    """ras_options.  Kernel-variant switches (same recurrences, summation order aside):
    fuse_p: fuse the PCG p update into the next SpMV (tiled path);
    plain: force FP64/int32 SELL instead of the default lane-packed SELL-Z;
    stage: shared-memory staging of p in the tiled SpMV;
    path: local-PCG execution path, "auto" | "tiled" | "block" | "resident" (ras_pcg_path);
    tiled: shorthand for path="tiled";
    robin: ORAS transmission parameter in [0, 1) (0 = RAS; ras_options.robin, R30).
    Other ras_options fields pass through **kw, e.g. async_persistent=0|1|2 (async driver,
    R33), detector, max_resumes, poll_interval, async_timeout_s."""
    o = F.RasOptions()
    _check(F.lib().ras_options_default(C.byref(o)))
    o.fuse_p = 1 if fuse_p else 0
    o.matrix_format = 1 if plain else 0
    o.stage_p = 1 if stage else 0
    o.pcg_path = _PATHS["tiled" if tiled else path]
    o.robin = float(robin)
    o.local_solver = _SOLVERS[local_solver] if isinstance(local_solver, str) else int(local_solver)
    o.inner_iters = int(inner_iters)
    o.inner_tol = float(inner_tol)
    o.detector = _DETECTORS[detector] if isinstance(detector, str) else int(detector)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class Plan:
    """Host-side setup plan (ras_plan.h): overlap sets and index maps, no GPU."""

    def __init__(self, A, b, owner, overlap, rank=0, world=1, num_subdomains=None, sub_to_rank=None):
        L = F.lib()
        self._csr, self._keep = _csr_struct(A)
        self._part, self._keep2 = _partition_struct(owner, num_subdomains, sub_to_rank)
        self._b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        h = C.c_void_p()
        _check(L.ras_plan_build(C.byref(h), C.byref(self._csr), F.ptr(self._b, F.F64), C.byref(self._part),
                                int(overlap), int(rank), int(world)))
        self._h = h
        self.rank, self.world = rank, world

    @classmethod
    def _borrow(cls, handle, owner_obj):
        self = cls.__new__(cls)
        self._h = handle
        self._owner_obj = owner_obj
        self._borrowed = True
        return self

    def __del__(self):
        if getattr(self, "_h", None) and not getattr(self, "_borrowed", False):
            F.lib().ras_plan_free(self._h)
            self._h = None

    def info(self) -> dict:
        i = F.RasPlanInfo()
        _check(F.lib().ras_plan_get_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def halo_request(self, src_rank):
        cnt, off = F.I64(), F.I64()
        _check(F.lib().ras_plan_halo_request(self._h, src_rank, C.byref(cnt), None, C.byref(off)))
        g = np.empty(cnt.value, dtype=np.int64)
        _check(F.lib().ras_plan_halo_request(self._h, src_rank, C.byref(cnt), F.ptr(g, F.I64), C.byref(off)))
        return g, off.value

    def set_send(self, dst_rank, gids, remote_offset):
        g = np.ascontiguousarray(gids, dtype=np.int64)
        _check(F.lib().ras_plan_set_send(self._h, dst_rank, len(g), F.ptr(g, F.I64), int(remote_offset)))

    def finalize(self):
        _check(F.lib().ras_plan_finalize(self._h))

    def band_cholesky(self, local_idx):
        """ras_plan_band_cholesky: (L band (n, b+1), b) of local subdomain local_idx (after finalize)."""
        n, bw = F.I64(), F.I32()
        _check(F.lib().ras_plan_band_cholesky(self._h, int(local_idx), C.byref(n), C.byref(bw), None))
        out = np.empty((n.value, bw.value + 1), dtype=np.float64)
        _check(F.lib().ras_plan_band_cholesky(self._h, int(local_idx), C.byref(n), C.byref(bw), F.ptr(out, F.F64)))
        return out, bw.value

    def set_robin(self, robin):
        _check(F.lib().ras_plan_set_robin(self._h, float(robin)))

    def comm_pattern(self) -> np.ndarray:
        """ras_plan_comm_pattern: P x P receive counts, row = receiver (Fig. 2), this rank's rows."""
        P = self.info()["num_subdomains"]
        out = np.empty((P, P), dtype=np.int64)
        _check(F.lib().ras_plan_comm_pattern(self._h, F.ptr(out, F.I64)))
        return out

    def subdomain(self, local_idx):
        p, no, ng = F.I32(), F.I64(), F.I64()
        _check(F.lib().ras_plan_subdomain(self._h, local_idx, C.byref(p), C.byref(no), None, None, C.byref(ng), None))
        om = np.empty(no.value, np.int64)
        ow = np.empty(no.value, np.uint8)
        gh = np.empty(ng.value, np.int64)
        _check(F.lib().ras_plan_subdomain(self._h, local_idx, C.byref(p), C.byref(no), F.ptr(om, F.I64),
                                          F.ptr(ow, F.U8), C.byref(ng), F.ptr(gh, F.I64)))
        return p.value, om, ow.astype(bool), gh

    def maps(self, local_idx):
        _, om, _, gh = self.subdomain(local_idx)
        rs = np.empty(len(om), np.int32)
        ps = np.empty(len(om), np.int32)
        gs = np.empty(len(gh), np.int32)
        _check(F.lib().ras_plan_maps(self._h, local_idx, F.ptr(rs, F.I32), F.ptr(ps, F.I32), F.ptr(gs, F.I32)))
        return rs, ps, gs

    def send_list(self, dst_rank):
        cnt, off = F.I64(), F.I64()
        _check(F.lib().ras_plan_send_list(self._h, dst_rank, C.byref(cnt), None, None, C.byref(off)))
        g = np.empty(cnt.value, np.int64)
        s = np.empty(cnt.value, np.int32)
        _check(F.lib().ras_plan_send_list(self._h, dst_rank, C.byref(cnt), F.ptr(g, F.I64), F.ptr(s, F.I32),
                                          C.byref(off)))
        return g, s, off.value

    def storage_gids(self):
        i = self.info()
        own = np.empty(i["n_own"], np.int64)
        halo = np.empty(i["n_halo"], np.int64)
        _check(F.lib().ras_plan_storage_gids(self._h, F.ptr(own, F.I64), F.ptr(halo, F.I64)))
        return own, halo


class Solver:
    """One rank's RAS context (ras_setup ... ras_free).

    A: full CSR (ras_inputs.CSR / scipy) or a row window with .row0 / .n.
    b: RHS for the same rows as A.  owner: len-n owner array.
    comm: None (1 GPU) or dict(rank, world, device, nccl_id=bytes, stream=int, transport="nccl"|"loopback").
    Loopback (ras_comm.transport): `world` virtual ranks on one device, one host thread per
    rank; nccl_id is then any 128-byte group key shared by the group's ranks.
    """

    def __init__(self, A, b, owner, overlap, opts=None, comm=None, num_subdomains=None, sub_to_rank=None):
        L = F.lib()
        csr, keep = _csr_struct(A)
        part, keep2 = _partition_struct(owner, num_subdomains, sub_to_rank)
        b = np.ascontiguousarray(b, dtype=np.float64)
        self.n = csr.n
        o = opts if opts is not None else options()
        cm = None
        self._id = None
        if comm is not None:
            cm = F.RasComm()
            cm.rank, cm.world, cm.device = int(comm.get("rank", 0)), int(comm.get("world", 1)), int(comm.get("device", 0))
            if comm.get("nccl_id") is not None:
                self._id = C.create_string_buffer(bytes(comm["nccl_id"]), 128)
                cm.nccl_unique_id = C.cast(self._id, C.c_void_p)
            cm.cuda_stream = comm.get("stream") or None
            cm.transport = F.RAS_TRANSPORT_LOOPBACK if comm.get("transport") == "loopback" else F.RAS_TRANSPORT_NCCL
            self.rank, self.world = cm.rank, cm.world
        else:
            self.rank, self.world = 0, 1
        h = C.c_void_p()
        _check(L.ras_setup(C.byref(h), C.byref(csr), F.ptr(b, F.F64), C.byref(part), int(overlap), C.byref(o),
                           C.byref(cm) if cm is not None else None))
        self._h = h
        del keep, keep2

    def close(self):
        if getattr(self, "_h", None):
            F.lib().ras_free(self._h)
            self._h = None

    __del__ = close

    def set_rhs(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        _check(F.lib().ras_set_rhs(self._h, F.ptr(b, F.F64)), self._h)

    def solve(self, tol=1e-8, max_iters=10000, mode="sync", x0=None, gather=True, raise_on_noconv=False):
        """Returns (status, x or None).  status RAS_OK / RAS_ENOCONV / RAS_EVERIFY."""
        md = F.RAS_SYNC if mode == "sync" else F.RAS_ASYNC
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.empty(self.n, dtype=np.float64) if gather else None
        st = F.lib().ras_solve(self._h, float(tol), int(max_iters), md, F.ptr(x0a, F.F64), F.ptr(x, F.F64))
        if st not in (F.RAS_OK, F.RAS_ENOCONV, F.RAS_EVERIFY) or (raise_on_noconv and st != F.RAS_OK):
            _check(st, self._h)
        return st, x

    def solve_device(self, tol, max_iters, mode="sync", x0_ptr=None, x_ptr=None):
        md = F.RAS_SYNC if mode == "sync" else F.RAS_ASYNC
        st = F.lib().ras_solve_device(self._h, float(tol), int(max_iters), md, x0_ptr, x_ptr)
        if st not in (F.RAS_OK, F.RAS_ENOCONV, F.RAS_EVERIFY):
            _check(st, self._h)
        return st

    def stats(self) -> dict:
        s = F.RasStats()
        _check(F.lib().ras_stats(self._h, C.byref(s)), self._h)
        return s.as_dict()

    def owned_gids(self) -> np.ndarray:
        n = F.lib().ras_owned_count(self._h)
        g = np.empty(n, np.int64)
        _check(F.lib().ras_owned_gids(self._h, F.ptr(g, F.I64)), self._h)
        return g

    def update_counts(self) -> np.ndarray:
        nl = self.plan().info()["local_subdomains"]
        out = np.empty(nl, np.int64)
        _check(F.lib().ras_update_counts(self._h, F.ptr(out, F.I64)), self._h)
        return out

    def plan(self) -> Plan:
        h = C.c_void_p()
        _check(F.lib().ras_ctx_plan(self._h, C.byref(h)), self._h)
        return Plan._borrow(h, self)

    def kernel_timing(self, enable=True):
        _check(F.lib().ras_kernel_timing(self._h, 1 if enable else 0), self._h)

    def kernel_times(self) -> dict:
        """{name: (launches, total_ms, bytes_per_launch)} of the last solve."""
        arr = (F.RasKernelTime * 16)()
        n = F.I32()
        _check(F.lib().ras_kernel_times(self._h, arr, 16, C.byref(n)), self._h)
        return {arr[i].name.decode(): (arr[i].launches, arr[i].total_ms, arr[i].bytes_per_launch)
                for i in range(n.value)}

    def set_scripted_flags(self, flags):
        f = np.ascontiguousarray(flags, dtype=np.uint8)
        _check(F.lib().ras_set_scripted_flags(self._h, F.ptr(f, F.U8), f.shape[0]), self._h)

    def put_stress(self, epochs, words) -> dict:
        """ras_debug_put_stress (collective, world == 2): torn / stale words seen by rank 1."""
        out = np.zeros(4, np.int64)
        _check(F.lib().ras_debug_put_stress(self._h, int(epochs), int(words), F.ptr(out, F.I64)), self._h)
        return dict(zip(("torn", "stale", "regress", "observations"), out.tolist()))

    def detector_stops(self) -> np.ndarray:
        nl = self.plan().info()["local_subdomains"]
        out = np.empty(nl, np.int64)
        _check(F.lib().ras_detector_stops(self._h, F.ptr(out, F.I64)), self._h)
        return out
