/*
 * ras.h — C ABI of the B200-native (a)synchronous Restricted Additive Schwarz
 * hot path (arxiv 2003.05361).  Plain C types only; no torch types.
 *
 * Citations: "P<n>" = PAPER.md line n (section / equation / algorithm named),
 * "S<n>" = SPEC.md line n, "R<n>" = reading n in DESIGN.md.
 *
 * What the library computes (PAPER §2.1, P114-153; Alg. 1, P233-245):
 *   the solution of A x = b (Eq. 1, P114-118), A sparse SPD, by RAS sweeps.
 *   One sweep, for every subdomain p (all run in this library's CUDA kernels):
 *     a1  restrict   x^k onto Omega_p u Gamma_p (owned / halo storage)
 *     a2  residual   r~_p = b~_p - A_p x[Omega_p] - B_p x[Gamma_p]   (P292-297)
 *     a3  local solve A_p d = r~_p  (Jacobi-PCG, IC(0)/ILU(0)-PCG, P309-323)
 *     a4  restricted prolongation x^{k+1}[S_p] = x^k[S_p] + d[S_p]  (P147-153)
 *     a5  exchange of the owner values other subdomains need       (P359-397)
 *     a6  convergence: global ||b-Ax|| < tau ||b|| (sync, P344-346) or
 *         Eq. 2 local flags + centralized / decentralized detection (async,
 *         P326-357), verified after termination (P346-348).
 *
 * Conventions (all functions):
 *   - Every input pointer is BORROWED for the duration of the call only; the
 *     library copies what it needs (host -> device).  Host pointers unless
 *     stated otherwise.
 *   - Indices are 0-based.  FP64 values (R16: the paper states no precision).
 *   - A context (ras_ctx) owns every device buffer it allocates and is NOT
 *     thread-safe.  ras_setup / ras_solve are COLLECTIVE over the ranks of a
 *     multi-GPU run: every rank calls them with identical tol, mode, overlap,
 *     partition and options.
 *   - Errors are returned as ras_status; ras_last_error() gives the message.
 *     A NULL context or argument where one is required returns RAS_EINVAL.
 */
#ifndef RAS_H_
#define RAS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAS_ABI_VERSION 4

typedef struct ras_ctx ras_ctx; /* opaque; one per rank (process) */

typedef enum {
  RAS_OK = 0,
  RAS_EINVAL = 1,   /* bad argument: dims, unsorted/out-of-range columns, owner out of range,
                       empty subdomain, overlap < 0, tol <= 0, row window too small (S42) */
  RAS_ENOTSPD = 2,  /* non-positive diagonal or IC(0)/ILU(0) pivot; message names the subdomain (S480) */
  RAS_ENOCONV = 3,  /* max_iters reached; x_out holds the last iterate, stats valid (S78, S498) */
  RAS_EVERIFY = 4,  /* async terminated but ||b-Ax|| >= tau ||b|| after max_resumes (S507, R20) */
  RAS_ECUDA = 5,    /* CUDA runtime error (text passed through) */
  RAS_ENCCL = 6,    /* NCCL error (text passed through) */
  RAS_ENOMEM = 7,   /* host or device allocation failed */
  RAS_ESTATE = 8    /* call not valid in the current state (e.g. no GPU, NCCL missing for world>1) */
} ras_status;

typedef enum { RAS_SYNC = 0, RAS_ASYNC = 1 } ras_mode;

typedef enum {
  RAS_LS_JACOBI_PCG = 0, /* PCG, M = diag(A_p), fixed m iterations (P313-315; R6, R8) */
  RAS_LS_IC0_PCG = 1,    /* PCG, M = L L^T, IC(0) of A_p, level-scheduled trisolves (P317-323; R9).
                            Trisolve kernel (same products in the same order):
                            one thread-block cluster per subdomain walking its levels, dependencies
                            pushed through distributed shared memory (k_trsv_ds), when every
                            dependency lies in the previous level and rows have <= 4 dependencies /
                            consumers; else the cluster walk through L2 (k_trsv_cl) when the levels
                            fit its clusters; else chunks over the whole GPU, each waiting for the
                            chunks it depends on (k_trsv_pf; rows with <= 4 dependencies) or for
                            the previous level (k_trsv).  Environment RAS_TRSV=cl|pf|level|sf
                            forces k_trsv_cl / k_trsv_pf / k_trsv / the sync-free k_trsv_sf */
  RAS_LS_ILU0_PCG = 2,   /* PCG, M = L U, ILU(0) of A_p (R10) */
  RAS_LS_EXACT_PCG = 3,  /* Jacobi-PCG to ||r|| <= 1e-14 ||r~||, <= 10|Omega_p| iterations:
                            the iterative stand-in for the paper's direct local solve (P317-318; R6) */
  RAS_LS_CHOLESKY = 4    /* direct local solve (P311-318, NEXT f1): complete Cholesky factor of A_p in
                            natural Omega_p order (banded, computed on the host once in ras_setup),
                            two banded triangular solves per local solve, one CTA per subdomain.
                            Needs every padded |Omega_p| <= 12288 rows and the bands (2 n (b+1) FP64
                            per subdomain) <= 16 GB in total, else RAS_EINVAL; RAS_ENOTSPD on a
                            non-positive pivot */
} ras_local_solver;

typedef enum { RAS_DET_CENTRAL = 0, RAS_DET_DECENTRAL = 1 } ras_detector;

/* How the Jacobi / exact local PCG (a3) is executed on the GPU.  All paths run
 * the same recurrences; only the summation order of the dot
 * products differs.  IC(0)/ILU(0) always use TILED.
 *   TILED    one streaming launch per PCG pass over every subdomain's rows
 *   BLOCK    one CTA per subdomain runs the whole local solve in shared memory
 *            (|Omega_p| <= 14336 padded rows; the paper's 4096-unknown regime)
 *   RESIDENT a cooperative grid, one CTA per SM, runs each subdomain's whole
 *            local solve with p, r, d in shared memory and q in registers
 *            (a chunk of <= kResidMaxRPT * 768 rows per CTA of its group).  Sync
 *            solves run every local subdomain in one launch; async solves issue
 *            one launch per two consecutive subdomains' updates (its two lanes),
 *            one pair after another (R34; RAS_ASYNC_PAIRS=0: singly)
 *   AUTO     BLOCK if it applies, else RESIDENT if it applies, else TILED */
typedef enum { RAS_PCG_AUTO = 0, RAS_PCG_TILED = 1, RAS_PCG_BLOCK = 2, RAS_PCG_RESIDENT = 3 } ras_pcg_path;

/* Sparse matrix A in CSR, possibly a window of rows [row_begin, row_begin+nrows)
 * of the global n x n matrix (so a rank need not hold all of A).  row_ptr is
 * relative: row_ptr[0] == 0, row_ptr[nrows] == nnz of the window.  Columns are
 * global, strictly increasing within a row, in [0, n).  A rank's window must
 * contain every row of its subdomains' Omega_p (else RAS_EINVAL). */
typedef struct {
  int64_t n;
  int64_t row_begin;
  int64_t nrows;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
} ras_csr;

/* Non-overlapping partition (PAPER §3.2.1, P247-290): owner[g] in [0, P) is the
 * subdomain owning global row g (len n, full on every rank).  sub_to_rank[p]
 * maps subdomains to ranks (GPUs); NULL = contiguous blocks
 * (rank r gets p in [r*P/world, (r+1)*P/world)). */
typedef struct {
  int32_t num_subdomains;
  const int32_t* owner;
  const int32_t* sub_to_rank;
} ras_partition;

typedef struct {
  ras_local_solver local_solver; /* default RAS_LS_JACOBI_PCG */
  int32_t inner_iters;           /* m (default 20); ignored by EXACT */
  double inner_tol;              /* eta: stop the local PCG when ||r|| <= eta ||r~|| (0 = fixed m) */
  ras_detector detector;         /* async termination detection (default DECENTRAL, P481-484) */
  int32_t local_crit_owned_only; /* Eq. 2 over owned rows only (R12); default 0 = paper's Eq. 2 */
  int32_t max_resumes;           /* async: resumes after failed verification (R20), default 3 */
  int32_t use_graphs;            /* async stream driver, fixed-m local solves: replay each subdomain's
                                    update as a captured CUDA graph (default 1) */
  int32_t poll_interval;         /* sweeps between host polls of the device stop flag (default 4) */
  double async_timeout_s;        /* async wall-clock watchdog, default 1800 s */
  int32_t scripted_flags;        /* test hook: Eq. 2 flags come from ras_set_scripted_flags */
  /* kernel variants (bitwise-equivalent results up to summation order) */
  int32_t fuse_p;                /* 1: fuse the PCG p update into the next SpMV (tiled path, plain SELL) */
  int32_t matrix_format;         /* 0: lane-packed SELL-Z when the matrix allows it; 1: plain SELL-32 */
  int32_t stage_p;               /* 1: stage p in shared memory in the tiled SpMV */
  ras_pcg_path pcg_path;         /* default RAS_PCG_AUTO */
  int32_t async_persistent;      /* async on one or more GPUs with BLOCK-sized subdomains: one persistent
                                    cooperative kernel per GPU, every CTA iterating its subdomains with no
                                    host involvement.  2 (default) = for tolerance-based local solves
                                    (exact / inner_tol > 0) and, on one GPU, for fixed-m PCG too, whose
                                    residuals there read every neighbour's update whole (per-subdomain
                                    sequence counters: without them fixed-m PCG diverges on thin strips,
                                    R33; environment RAS_PERSISTENT_SEQLOCK=0 turns them off);
                                    1 = always; 0 = CUDA streams */
  int32_t force_first_stop;      /* test hook (async): in the first detection round every Eq. 2 flag reads
                                    as set, so detection terminates after a few updates and the
                                    post-termination verification fails -> the R20 resume path runs */
  int32_t persistent_grid;       /* persistent async kernel: at most this many CTAs (0 = one per subdomain up to
                                    the co-resident limit).  1 = ONE CTA updating every subdomain in turn, each
                                    update reading the latest x: the sequential schedule the oracle's
                                    ras_schedule reproduces (parity hook for the persistent kernel) */
  /* Optimized RAS (NEXT f3, PAPER P760-763, R30): Robin-type transmission condition in algebraic
   * form -- the local solve uses A~_p = A_p - robin * diag(sum_{j not in Omega_p} |a_ij|) (rows
   * coupled outside Omega_p); the residual keeps A.  0 = RAS (Dirichlet truncation, default);
   * -> 1 approaches Neumann.  Must be in [0, 1) (A~_p stays SPD) and > 0 needs overlap >= 1
   * (the restricted iteration diverges without overlap), else RAS_EINVAL. */
  double robin;
  double reserved_d[3];
  int32_t device_setup;          /* 1 (default): the gamma-hop overlap sets Omega_p / Gamma_p, the owned and
                                    halo slot maps and the receive counts are built by CUDA kernels
                                    (row a0 on the device); 0: by the host BFS of the plan (ras_plan.h).
                                    Both give identical plans (bit-exact, tested) */
  int32_t reserved_j[3];
} ras_options;

/* Transport of a multi-rank context (ras_comm.transport). */
typedef enum {
  RAS_TRANSPORT_NCCL = 0,     /* one process per GPU: NCCL collectives + CUDA IPC peer windows over NVLink */
  RAS_TRANSPORT_LOOPBACK = 1  /* test transport: `world` virtual ranks driven by host threads of ONE process
                                 on ONE device.  Collectives are host rendezvous of the group's threads
                                 (device buffers staged through the host or copied device-to-device); peer
                                 windows are the peers' plain device pointers, so the async kernels' puts,
                                 version counters and detector boards run unchanged.  Every rank's thread
                                 must call ras_setup / ras_solve / ras_set_rhs concurrently (they are
                                 collective); a rank that never arrives makes the others fail with
                                 RAS_ESTATE after 600 s instead of hanging. */
} ras_transport;

/* Multi-GPU plumbing.  NULL = single GPU (current device, default stream). */
typedef struct {
  int32_t rank, world;          /* this process's rank and the number of ranks (GPUs) */
  int32_t device;               /* CUDA device ordinal this rank drives */
  const void* nccl_unique_id;   /* 128 bytes from ras_nccl_unique_id() on rank 0, broadcast by
                                   the caller (torch.distributed); NULL when world == 1.  LOOPBACK:
                                   any 128 bytes naming the group, identical on its ranks */
  void* cuda_stream;            /* cudaStream_t for sync-mode work; NULL = a library stream */
  /* optional device allocator hooks (e.g. torch's caching allocator); NULL = cudaMalloc */
  void* (*dev_alloc)(size_t bytes, void* user);
  void (*dev_free)(void* ptr, void* user);
  void* alloc_user;
  int32_t transport;            /* ras_transport (0 = NCCL) */
} ras_comm;

typedef struct {
  int32_t mode, converged, verified, resumes;
  double time_to_solution_s;   /* start of ras_solve -> stop observed (R26; P474-480) */
  double setup_s;              /* ras_setup wall time (untimed by the paper, P229-231) */
  double verify_s;             /* gather + true residual after async stop */
  int64_t sweeps;              /* sync: global sweeps performed; async: max per-subdomain updates */
  int64_t updates_min, updates_median, updates_max; /* per-subdomain local solves (Fig. 7c, P727-735) */
  int64_t inner_iters_total;   /* total local PCG iterations over all subdomains on this rank */
  double final_rel_residual;   /* true ||b - A x|| / ||b|| of the returned iterate */
  /* per-phase device seconds of the last solve (Figs. 3a-7a: restrict + residual, local solve, prolongation,
   * exchange, convergence check).  Sync: CUDA events around each batched phase on the library stream
   * (every local subdomain advances together, so this is also each subdomain's time); their sum is the
   * device part of time_to_solution_s.  Async: %globaltimer at the phase boundaries of every update,
   * summed over a subdomain's updates and averaged over the local subdomains.  Where the local solve
   * kernel also prolongs (BLOCK, RESIDENT, direct) t_prolong is 0 and the prolongation is in t_local_solve. */
  double t_residual, t_local_solve, t_prolong, t_exchange, t_convcheck;
  double model_bytes;          /* algorithmic HBM bytes moved by this rank's kernels */
  int32_t num_subdomains, world;
  int32_t local_subdomains;
  int32_t pcg_path;            /* ras_pcg_path the local solves of the last solve ran on (sync or async) */
  int64_t rows_local;          /* sum |Omega_p| on this rank */
  int64_t halo_values;         /* halo slots on this rank (values received per exchange) */
  int64_t kernel_launches;     /* kernels launched by the last ras_solve on this rank */
  int64_t fresh_halo_reads;    /* async: halo version changes observed */
  int32_t resident_pattern;    /* RESIDENT path: 1 = row-pattern dictionary SpMV, 0 = SELL-Z / SELL stream */
  int32_t resident_lanes;      /* RESIDENT path: 0 = k_resident_pcg (r, d in shared memory); 1 / 2 =
                                  k_resident2 (r, d in tensor memory) with that many subdomains per CTA */
} ras_stats_t;

/* Fill *opt with defaults. */
ras_status ras_options_default(ras_options* opt);

/* Alg. 1 `initialization_and_setup` (P233-237): validate; partition bookkeeping;
 * gamma-hop overlap Omega_p and ghosts Gamma_p (P133-142, R1); restrict /
 * prolong / pack index maps; batched local matrices on the device; optional
 * IC(0)/ILU(0) factors and level sets; NCCL communicator and peer windows.
 * b: RHS rows for the same window as A (len A->nrows).  overlap = gamma >= 0.
 * On failure *out is NULL and ras_last_error(NULL) holds the message. */
ras_status ras_setup(ras_ctx** out, const ras_csr* A, const double* b, const ras_partition* part,
                     int32_t overlap, const ras_options* opt, const ras_comm* comm);

/* Replace the right-hand side (same window as at setup). */
ras_status ras_set_rhs(ras_ctx* ctx, const double* b);

/* Alg. 1 `solve` (P238-244).  tol = tau > 0.  max_iters: sync = sweeps,
 * async = per-subdomain updates (R21).  x0: host, len n (NULL = 0, R15).
 * x_out: host, len n, the gathered solution (owner values, P242) on every
 * rank, or NULL.  Returns RAS_OK, RAS_ENOCONV (x_out = x^{max_iters}; the
 * parity hook: max_iters = k returns the k-th sync iterate), RAS_EVERIFY, or
 * an error.  Sync mode stops at the first k with ||b - A x^k|| < tau ||b||
 * and returns x^k (R13). */
ras_status ras_solve(ras_ctx* ctx, double tol, int64_t max_iters, ras_mode mode, const double* x0,
                     double* x_out);

/* Distributed variant: x0 / x_out hold only THIS rank's owned values (len
 * ras_owned_count(), ordered as ras_owned_gids()), as device pointers or host
 * pointers (pinned or pageable; unified addressing picks the copy direction);
 * either may be NULL.  No global gather: every rank moves n_own values, so the
 * host<->device traffic of a solve does not grow with the number of GPUs. */
ras_status ras_solve_device(ras_ctx* ctx, double tol, int64_t max_iters, ras_mode mode, const double* x0_owned_dev,
                            double* x_owned_dev);

int64_t ras_owned_count(const ras_ctx* ctx);
/* Global ids of this rank's owned values in storage order (len ras_owned_count). */
ras_status ras_owned_gids(const ras_ctx* ctx, int64_t* gids_out);

ras_status ras_stats(const ras_ctx* ctx, ras_stats_t* out);

/* Per-subdomain update counts of the last solve (len = local subdomains). */
ras_status ras_update_counts(const ras_ctx* ctx, int64_t* counts_out);

void ras_free(ras_ctx* ctx);

/* Message of the last failure on ctx; ctx == NULL -> thread-local message of the
 * last failed ras_setup / ras_partition_regular / plan call.  Never NULL. */
const char* ras_last_error(const ras_ctx* ctx);

/* Regular block partition (regular1d / regular2d / 3D blocks, P277-286; R23):
 * nx*ny*nz grid, point (x,y,z) -> (z*ny+y)*nx+x; px*py*pz blocks whose sizes
 * differ by <= 1 per axis, earlier blocks larger; id = (bz*py+by)*px+bx.
 * owner_out: len nx*ny*nz.  RAS_EINVAL if a block would be empty. */
ras_status ras_partition_regular(int32_t nx, int32_t ny, int32_t nz, int32_t px, int32_t py, int32_t pz,
                                 int32_t* owner_out);

/* NCCL unique id (128 bytes) for multi-GPU setup; call on rank 0 only. */
ras_status ras_nccl_unique_id(void* out128);

/* Test hook (options.scripted_flags = 1): the Eq. 2 flag of local subdomain i in
 * sweep k is flags[k * nlocal + i] (k >= nsweeps -> last row). */
ras_status ras_set_scripted_flags(ras_ctx* ctx, const uint8_t* flags, int64_t nsweeps);

/* Debug / stress test of the one-sided put path (reading R17: 8-byte single-copy
 * atomicity of remote stores + release-published versions; P389-397).  COLLECTIVE
 * over a world == 2 context: rank 0 writes `epochs` epochs of `words` epoch-tagged
 * 8-byte words into rank 1's x window (the stores the async puts use), each
 * followed by a system-scope fence + version increment; rank 1 polls the version
 * (acquire) and checks the window after every observation.  out4 (rank 1):
 * {torn words, stale words, version regressions, observations}; zeros on rank 0.
 * words <= the reader's storage (owned + halo).  Destroys both ranks' iterate. */
ras_status ras_debug_put_stress(ras_ctx* ctx, int64_t epochs, int64_t words, int64_t* out4);

/* Per-subdomain stop sweep of the last scripted run (len local subdomains). */
ras_status ras_detector_stops(const ras_ctx* ctx, int64_t* stop_out);

/* Per-kernel CUDA-event timing on the library stream (for the roofline report).
 * When enabled, every kernel launch of ras_solve* on the library stream is
 * bracketed by events (sync mode; the async drivers' per-subdomain streams and
 * graphs are not timed); the totals of the last solve are returned per kernel
 * kind: k_residual, k_spmv_dot, k_update_dot, k_pupdate, k_prolong, k_pack,
 * control (scalar / check kernels), k_trsv, k_zdot, k_small_pcg (BLOCK),
 * k_resident_pcg (RESIDENT), k_band_chol (direct solve).  bytes_per_launch is
 * the DESIGN.md §5 model; for the whole-solve kernels (BLOCK / RESIDENT) it is the
 * compulsory HBM bytes of one launch.  out may be NULL to query the count. */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;          /* sum of event-measured launch durations */
  double bytes_per_launch;  /* algorithmic HBM bytes of one launch */
} ras_kernel_time_t;

ras_status ras_kernel_timing(ras_ctx* ctx, int32_t enable);
ras_status ras_kernel_times(const ras_ctx* ctx, ras_kernel_time_t* out, int32_t max_entries, int32_t* n_out);

int32_t ras_abi_version(void);

/* Hash of the sources, headers, defines and flags this library was built from
 * (paper_2003_05361_b200/build.py); the Python binding refuses a library whose
 * hash differs from the tree it is loaded from.  Static string, never NULL. */
const char* ras_build_hash(void);

#ifdef __cplusplus
}
#endif

#endif /* RAS_H_ */
