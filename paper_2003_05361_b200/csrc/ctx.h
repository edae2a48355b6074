// ras_ctx: one per rank.  Owns the plan, every device buffer, streams, NCCL.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "plan_internal.h"
#include "ras.h"

namespace ras {

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool raw = false;  // cudaMalloc'd IPC-capable window (never through the allocator hook)
};

struct AsyncRt;    // async-mode runtime (async.cu)
struct LoopGroup;  // loopback transport group (comm.cu)

// one side of a point-to-point transfer (device buffer, element count)
struct Xfer {
  int peer;
  void* buf;
  size_t count;
};

enum KId { K_RES = 0, K_SPMV, K_UPD, K_PUPD, K_PROL, K_PACK, K_CTRL, K_TRSV, K_ZDOT, K_SMALL, K_RESID, K_BAND, K_NKINDS };

// A range of tiles: every local subdomain (lp < 0) or one subdomain.
struct Range {
  int64_t tile_base;
  unsigned ntiles;
  int lp;        // first local subdomain, -1 = all
  int nsub = 1;  // subdomains from lp (consecutive; RESIDENT / scalar kernels)
};

// Device copy of one level-ordered triangular factor (factor.cpp / k_trsv).
struct TriBuf {
  TriDev dev{};
  int32_t nchunks = 0;
  int32_t nlev_slots = 0;  // size of the per-(subdomain, level) done counters
  std::vector<int32_t> sub_c0, sub_nc, sub_lev_off, sub_nlev;
  int32_t* d_lev_done = nullptr;
  double bytes = 0.0;      // algorithmic bytes of one solve
  // cluster-resident solve (k_trsv_cl): position-ordered ELL copy, only when every
  // row has <= 4 dependencies
  bool cl_ok = false;
  TriCl cl{};
  std::vector<int32_t> sub_max_lev;  // rows of the largest level per subdomain
  // DSMEM-routed solve (k_trsv_ds): routing tables for cluster size ds_ncl
  int2* d_cdep = nullptr;     // k_trsv_pf: per chunk, the range of chunk ids its rows depend on
  int32_t* d_cflag = nullptr;  // k_trsv_pf: per chunk, 1 once completed in the current launch
  bool ds_ok = false;
  int ds_ncl = 0;
  TriDs ds{};
};

struct KTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<int32_t> kind;  // per recorded pair
  size_t used = 0;            // events used in this solve
  double total_ms[K_NKINDS] = {};
  int64_t count[K_NKINDS] = {};
};

struct ModelBytes {  // algorithmic bytes per launch over the whole row space
  double residual, spmv_dot, update_dot, pupdate, prolong, pack, trsv, zdot;
  double local_solve;  // BLOCK / RESIDENT: compulsory HBM bytes of one whole local-solve launch
  double band;         // direct solve: both bands read once + r~ in + x[S_p] read/written
};

}  // namespace ras

struct ras_ctx {
  ras_plan* plan = nullptr;
  ras_options opt{};
  int32_t rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t nccl = nullptr;
  std::shared_ptr<ras::LoopGroup> loop;  // loopback transport (ras_comm.transport); null = NCCL
  std::string loop_key;
  bool loopback = false;
  void* (*dev_alloc)(size_t, void*) = nullptr;
  void (*dev_free)(void*, void*) = nullptr;
  void* alloc_user = nullptr;
  std::vector<ras::DevBuf> bufs;
  std::string err;
  double setup_s = 0.0;
  double setup_phase[4] = {};  // plan, finalize, upload + layouts, async runtime (RAS_SETUP_TRACE)
  double b2_global = 0.0;  // ||b||^2

  // ---- device arrays ----
  int64_t rows_pad = 0, n_own = 0, n_halo = 0, ntiles = 0;
  int32_t nl = 0;  // local subdomains
  double* d_b = nullptr;
  double* d_diag = nullptr;
  int32_t* d_own_slot = nullptr;
  ras::Sell R{}, L{};
  int wR = 0, wL = 0;  // widest SELL slice of each matrix (kernel width dispatch)
  bool z = false;      // SELL-Z compressed matrices + diagonal on the device
  int zwR = 0, zwL = 0;  // SELL-Z packed widths
  ras::Diag D{};
  ras::Tiles T{};
  int2* d_cspan = nullptr;  // per tile {first column, span} of the local matrix (SpMV smem staging)
  int32_t dir = 0;  // tile walk direction of the last streaming launch
  double* d_x = nullptr;  // storage [owned | halo]
  double* d_r = nullptr;
  double* d_p = nullptr;
  double* d_p2 = nullptr;  // p double buffer (fused p update + SpMV)
  bool fuse_p = false;     // options.fuse_p: fuse pass 3 into the next pass 1
  bool stage = false;      // options.stage_p: shared-memory staging of p in the SpMV
  int path = RAS_PCG_TILED;  // local-PCG path of batched (sync) solves, ras_pcg_path
  bool small = false;      // path == BLOCK: one CTA per subdomain runs the whole local PCG (k_small_pcg)
  int small_nmax = 0;
  ras::SmallSubs SS{};
  // path == RESIDENT (k_resident_pcg): cooperative grid of ngroups * gs CTAs
  ras::ResidentCtl RC{};
  int resid_rpt = 0;        // rows-per-thread instantiation
  size_t resid_smem = 0;    // dynamic shared memory per CTA (p, r of the largest chunk)
  int resid_chunk = 0;      // rows per CTA of the largest subdomain
  int resid_glo = 0, resid_ghi = 0;  // widest ghost zones below / above a chunk (rows)
  bool resid_pat = false;   // row-pattern dictionary SpMV (no matrix stream)
  int resid_lanes = 0;      // 0: k_resident_pcg (v1); 1 / 2: k_resident2 with NL lanes (TMEM)
  bool resid_seq = false;   // async sequential schedule: per-subdomain calls use k_resident_pcg
  unsigned long long* d_resid_slots = nullptr;
  double* d_q = nullptr;
  double* d_d = nullptr;
  // direct local solve (NEXT f1): banded Cholesky factors, k_band_chol
  bool chol = false;
  ras::BandDev band{};
  size_t band_smem = 0;
  // IC(0)/ILU(0) path (a3')
  bool ic = false;
  double* d_z = nullptr;
  double* d_y = nullptr;    // forward-solve output of the sync-free trisolve
  int trsv_cl_max = 0;      // largest usable cluster size of k_trsv_cl (16 with the non-portable opt-in, else 8)
  int trsv_cl_force = 0;    // RAS_TRSV_CL: fixed cluster size (tests), 0 = sized to the widest level
  std::vector<int> trsv_cl_fit;  // co-resident clusters of k_trsv_cl per cluster size (-1 = not queried)
  int trsv_cl_nt = 512;    // RAS_TRSV_CL_NT: row-taking threads per CTA (tests)
  bool trsv_cl_forced = false;  // RAS_TRSV=cl / RAS_TRSV_CL: k_trsv_cl even for levels wider than its prefetch
  bool trsv_ds = false;     // DSMEM-routed solves (k_trsv_ds) for both factors
  int trsv_mode = 0;        // 0 = cluster kernels when usable (default), 1 = level counters (k_trsv), 2 = sync-free, 3 = k_trsv_pf
  bool trsv_sf = false;     // sync-free trisolve (k_trsv_sf, RAS_TRSV=sf); default k_trsv (level barriers)
  ras::TriBuf tri_f, tri_b;
  uint32_t* d_trsv_ctr = nullptr;  // [2][nl + 1] chunk counters (per subdomain + batched)
  ras::Scal S{};
  int64_t* d_inner_total = nullptr;
  // sync control
  int32_t* d_stop = nullptr;
  ras::SyncState* d_sync = nullptr;
  double* d_r2_local = nullptr;
  double* d_r2_global = nullptr;
  int32_t* d_nactive = nullptr;
  int32_t* h_stop = nullptr;       // mapped pinned
  int32_t* h_stop_dev = nullptr;   // device alias of h_stop
  int32_t* h_nactive = nullptr;    // pinned
  // exchange (sync, NCCL)
  int64_t n_send = 0;
  int32_t* d_send_slot = nullptr;
  double* d_sendbuf = nullptr;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;  // per peer

  // async runtime
  ras::AsyncRt* async = nullptr;

  // stats of the last solve
  ras_stats_t st{};
  std::vector<int64_t> updates;
  std::vector<int64_t> det_stops;
  ras::ModelBytes mb{};
  int64_t launches = 0;
  ras::KTimer kt;
  // device copies of the storage gids (x0 scatter / x_out gather on device)
  int32_t* d_own_gid = nullptr;
  int32_t* d_halo_gid = nullptr;
  double* d_xglob = nullptr;  // len n, allocated on first host-buffer solve
  // N-GPU gather: owned values allgathered in padded segments of gmax (ensure_xglob)
  int64_t gmax = 0;
  int32_t* d_gid_all = nullptr;  // [world * gmax] global id of every gathered slot (-1 = padding)
  double* d_gsend = nullptr;     // [gmax]
  double* d_grecv = nullptr;     // [world * gmax]

  std::vector<uint8_t> scripted;
  int64_t scripted_sweeps = 0;
};

namespace ras {
ras_status set_err(ras_ctx* c, ras_status s, const std::string& m);
ras_status cuda_err(ras_ctx* c, cudaError_t e, const char* what);
void* dalloc(ras_ctx* c, size_t bytes);
void* dalloc_raw(ras_ctx* c, size_t bytes);
void dfree(ras_ctx* c, void* p);
ras_status allow_smem(ras_ctx* c, const void* fn);  // dynamic smem cap = device maximum
// collectives over the context's ranks (comm.cu): NCCL, or the loopback group
ras_status loop_join(ras_ctx* c, const void* key128);
void loop_leave(ras_ctx* c);
ras_status coll_allreduce(ras_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                          cudaStream_t s);
ras_status coll_allgather(ras_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t s);
ras_status coll_sendrecv(ras_ctx* c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, ncclDataType_t dt,
                         cudaStream_t s);
ras_status coll_allreduce_f64(ras_ctx* c, double* v, int n, bool is_max);  // host values, in place
ras_status coll_barrier(ras_ctx* c);  // device drained on every rank
ras_status solve_async(ras_ctx* c, double tol, int64_t max_iters);
int kt_begin(ras_ctx* c, cudaStream_t s);
void kt_end(ras_ctx* c, cudaStream_t s, int kind, int idx);
Range range_all(ras_ctx* c);
Range range_sub(ras_ctx* c, int lp);
ras_status enq_residual(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C);
ras_status enq_pcg(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C, int m, double inner_tol, bool exact);
ras_status enq_prolong(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C);
ras_status async_setup(ras_ctx* c);
ras_status async_set_b2(ras_ctx* c);  // re-upload the Eq. 2 ||b~_p||^2 after ras_set_rhs
void async_free(ras_ctx* c);
ras_status put_stress(ras_ctx* c, int64_t epochs, int64_t words, int64_t* out4);  // R17 stress test
ras_status plan_build_device(ras_ctx* c, ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part,
                             int32_t overlap);  // row a0 on the device (setup_dev.cu)
}  // namespace ras

#define TRY(x)                   \
  do {                           \
    ras_status s_ = (x);         \
    if (s_ != RAS_OK) return s_; \
  } while (0)

namespace ras {
template <class T>
inline ras_status upload(ras_ctx* c, T** dst, const std::vector<T>& src, size_t min_elems = 0) {
  size_t n = std::max(src.size(), min_elems);
  *dst = (T*)dalloc(c, n * sizeof(T));
  if (!*dst) return set_err(c, RAS_ENOMEM, "device allocation failed");
  // on the library stream (the one NCCL and the kernels use), completed before
  // return: the host vector may die and a collective may read *dst right away
  if (!src.empty() &&
      (cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
       cudaStreamSynchronize(c->stream) != cudaSuccess))
    return set_err(c, RAS_ECUDA, "cudaMemcpyAsync (upload) failed");
  return RAS_OK;
}

template <class T>
inline ras_status zalloc(ras_ctx* c, T** dst, size_t n) {
  *dst = (T*)dalloc(c, n * sizeof(T));
  if (!*dst) return set_err(c, RAS_ENOMEM, "device allocation failed");
  // stream-ordered before any later kernel / collective on the library stream
  if (cudaMemsetAsync(*dst, 0, std::max<size_t>(n, 1) * sizeof(T), c->stream) != cudaSuccess)
    return set_err(c, RAS_ECUDA, "cudaMemsetAsync failed");
  return RAS_OK;
}

// shared between the sync and async drivers (solver.cu)
ras_status sync_exchange(ras_ctx* c);                 // pack + NCCL send/recv into halo (a5, sync)
ras_status global_residual(ras_ctx* c, double* rel);  // true ||b - A x|| / ||b|| of the stored x
}  // namespace ras

#define RAS_CUDA(c, expr)                                         \
  do {                                                            \
    cudaError_t e_ = (expr);                                      \
    if (e_ != cudaSuccess) return ras::cuda_err((c), e_, #expr);  \
  } while (0)

#define RAS_NCCL(c, expr)                                                                        \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return ras::set_err((c), RAS_ENCCL, std::string(#expr ": ") + ncclGetErrorString(r_));     \
  } while (0)
