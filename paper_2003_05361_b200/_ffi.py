"""ctypes mirror of include/ras.h and include/ras_plan.h (argument marshalling only).

Loads the in-tree libras_b200.so and fails loudly if it is missing: there is no
CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RAS_LIB_PATH") or os.path.join(HERE, "libras_b200.so")

RAS_OK, RAS_EINVAL, RAS_ENOTSPD, RAS_ENOCONV, RAS_EVERIFY, RAS_ECUDA, RAS_ENCCL, RAS_ENOMEM, RAS_ESTATE = range(9)
STATUS_NAMES = ["RAS_OK", "RAS_EINVAL", "RAS_ENOTSPD", "RAS_ENOCONV", "RAS_EVERIFY", "RAS_ECUDA", "RAS_ENCCL",
                "RAS_ENOMEM", "RAS_ESTATE"]
RAS_SYNC, RAS_ASYNC = 0, 1
RAS_LS_JACOBI_PCG, RAS_LS_IC0_PCG, RAS_LS_ILU0_PCG, RAS_LS_EXACT_PCG, RAS_LS_CHOLESKY = range(5)
RAS_DET_CENTRAL, RAS_DET_DECENTRAL = 0, 1
RAS_PCG_AUTO, RAS_PCG_TILED, RAS_PCG_BLOCK, RAS_PCG_RESIDENT = range(4)
RAS_TRANSPORT_NCCL, RAS_TRANSPORT_LOOPBACK = 0, 1
ABI_VERSION = 4  # include/ras.h RAS_ABI_VERSION

I32, I64, F64, U8 = C.c_int32, C.c_int64, C.c_double, C.c_uint8
P = C.POINTER


class RasCsr(C.Structure):
    _fields_ = [("n", I64), ("row_begin", I64), ("nrows", I64), ("row_ptr", P(I64)), ("col_idx", P(I32)),
                ("val", P(F64))]


class RasPartition(C.Structure):
    _fields_ = [("num_subdomains", I32), ("owner", P(I32)), ("sub_to_rank", P(I32))]


class RasOptions(C.Structure):
    _fields_ = [("local_solver", I32), ("inner_iters", I32), ("inner_tol", F64), ("detector", I32),
                ("local_crit_owned_only", I32), ("max_resumes", I32), ("use_graphs", I32), ("poll_interval", I32),
                ("async_timeout_s", F64), ("scripted_flags", I32), ("fuse_p", I32), ("matrix_format", I32), ("stage_p", I32),
                ("pcg_path", I32), ("async_persistent", I32), ("force_first_stop", I32), ("persistent_grid", I32), ("robin", F64), ("reserved_d", F64 * 3),
                ("device_setup", I32), ("reserved_j", I32 * 3)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class RasComm(C.Structure):
    _fields_ = [("rank", I32), ("world", I32), ("device", I32), ("nccl_unique_id", C.c_void_p),
                ("cuda_stream", C.c_void_p), ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN),
                ("alloc_user", C.c_void_p), ("transport", I32)]


class RasStats(C.Structure):
    _fields_ = [("mode", I32), ("converged", I32), ("verified", I32), ("resumes", I32),
                ("time_to_solution_s", F64), ("setup_s", F64), ("verify_s", F64),
                ("sweeps", I64), ("updates_min", I64), ("updates_median", I64), ("updates_max", I64),
                ("inner_iters_total", I64), ("final_rel_residual", F64),
                ("t_residual", F64), ("t_local_solve", F64), ("t_prolong", F64), ("t_exchange", F64),
                ("t_convcheck", F64), ("model_bytes", F64), ("num_subdomains", I32), ("world", I32),
                ("local_subdomains", I32), ("pcg_path", I32), ("rows_local", I64), ("halo_values", I64),
                ("kernel_launches", I64), ("fresh_halo_reads", I64), ("resident_pattern", I32),
                ("resident_lanes", I32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RasPlanInfo(C.Structure):
    _fields_ = [("n", I64), ("num_subdomains", I32), ("rank", I32), ("world", I32), ("overlap", I32),
                ("local_subdomains", I32), ("tile_rows", I32), ("n_own", I64), ("n_halo", I64),
                ("rows_local", I64), ("rows_padded", I64), ("nnz_residual", I64), ("nnz_local", I64),
                ("sell_residual", I64), ("sell_local", I64), ("ntiles", I64), ("finalized", I32),
                ("z_format", I32)]


class RasKernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", I64), ("total_ms", F64), ("bytes_per_launch", F64)]


# (name, restype, argtypes) for every symbol declared in include/*.h
SIGNATURES = [
    ("ras_abi_version", I32, []),
    ("ras_build_hash", C.c_char_p, []),
    ("ras_options_default", I32, [P(RasOptions)]),
    ("ras_setup", I32, [P(C.c_void_p), P(RasCsr), P(F64), P(RasPartition), I32, P(RasOptions), P(RasComm)]),
    ("ras_set_rhs", I32, [C.c_void_p, P(F64)]),
    ("ras_solve", I32, [C.c_void_p, F64, I64, I32, P(F64), P(F64)]),
    ("ras_solve_device", I32, [C.c_void_p, F64, I64, I32, C.c_void_p, C.c_void_p]),
    ("ras_owned_count", I64, [C.c_void_p]),
    ("ras_owned_gids", I32, [C.c_void_p, P(I64)]),
    ("ras_stats", I32, [C.c_void_p, P(RasStats)]),
    ("ras_update_counts", I32, [C.c_void_p, P(I64)]),
    ("ras_free", None, [C.c_void_p]),
    ("ras_last_error", C.c_char_p, [C.c_void_p]),
    ("ras_partition_regular", I32, [I32, I32, I32, I32, I32, I32, P(I32)]),
    ("ras_nccl_unique_id", I32, [C.c_void_p]),
    ("ras_set_scripted_flags", I32, [C.c_void_p, P(U8), I64]),
    ("ras_detector_stops", I32, [C.c_void_p, P(I64)]),
    ("ras_debug_put_stress", I32, [C.c_void_p, I64, I64, P(I64)]),
    ("ras_kernel_timing", I32, [C.c_void_p, I32]),
    ("ras_kernel_times", I32, [C.c_void_p, P(RasKernelTime), I32, P(I32)]),
    # ras_plan.h
    ("ras_plan_build", I32, [P(C.c_void_p), P(RasCsr), P(F64), P(RasPartition), I32, I32, I32]),
    ("ras_plan_get_info", I32, [C.c_void_p, P(RasPlanInfo)]),
    ("ras_plan_halo_request", I32, [C.c_void_p, I32, P(I64), P(I64), P(I64)]),
    ("ras_plan_set_send", I32, [C.c_void_p, I32, I64, P(I64), I64]),
    ("ras_plan_finalize", I32, [C.c_void_p]),
    ("ras_plan_subdomain", I32, [C.c_void_p, I32, P(I32), P(I64), P(I64), P(U8), P(I64), P(I64)]),
    ("ras_plan_maps", I32, [C.c_void_p, I32, P(I32), P(I32), P(I32)]),
    ("ras_plan_send_list", I32, [C.c_void_p, I32, P(I64), P(I64), P(I32), P(I64)]),
    ("ras_plan_storage_gids", I32, [C.c_void_p, P(I64), P(I64)]),
    ("ras_plan_comm_pattern", I32, [C.c_void_p, P(I64)]),
    ("ras_plan_set_robin", I32, [C.c_void_p, F64]),
    ("ras_plan_band_cholesky", I32, [C.c_void_p, I32, P(I64), P(I32), P(F64)]),
    ("ras_plan_free", None, [C.c_void_p]),
    ("ras_ctx_plan", I32, [C.c_void_p, P(C.c_void_p)]),
]

_lib = None


def lib():
    """The loaded libras_b200.so (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.ras_abi_version() != ABI_VERSION:
            raise RuntimeError(f"{LIB_PATH} has ABI {L.ras_abi_version()}, the binding expects {ABI_VERSION}: rebuild it")
        if not os.environ.get("RAS_LIB_PATH"):  # explicit variant builds (tuning sweeps) skip the check
            from .build import source_hash

            want, have = source_hash(), L.ras_build_hash().decode()
            if have != want:
                raise RuntimeError(f"{LIB_PATH} was built from other sources (hash {have}, tree {want}): "
                                   "rebuild it with `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = L
    return _lib


class RasError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def ptr(a, ctype):
    return a.ctypes.data_as(P(ctype)) if a is not None else None
