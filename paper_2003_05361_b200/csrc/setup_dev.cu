// Row a0 on the device (round 2): the gamma-hop overlap construction and the
// index maps of one rank, built by CUDA kernels and handed to the host plan
// (plan.cpp) in exactly the form its host BFS produces, so everything after it
// (matrices, SELL / SELL-Z, factors) is shared and the two paths can be compared
// bit for bit (tests/test_gpu_setup.py).
//
// Definitions (PAPER §2.1 Fig. 1, P133-142; reading R1; include/ras_plan.h):
//   S_p      rows with owner[g] == p
//   Omega_p  S_p plus `overlap` breadth-first layers in the graph of A, ascending
//   Gamma_p  rows outside Omega_p adjacent to Omega_p, ascending
//   slot     owned rows: local subdomains ascending, each S_p ascending;
//            halo: every value of (Omega_p \ S_p) u Gamma_p of a local p owned by
//            another rank, deduplicated, sorted by (owning rank, gid)
// Kernels: one level array (int8) per subdomain over all n rows; round l marks the
// unvisited neighbours of the level-l rows with l + 1 (every writer of a row in a
// round writes the same value: the race is benign); rounds 0..gamma give Omega_p
// (levels <= gamma) and Gamma_p (level gamma + 1); stream compaction (CUB) in
// ascending gid order; scans for the slots; a per-subdomain histogram of owners
// over need_p for the receive counts (Fig. 2).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "ctx.h"
#include "plan_internal.h"

namespace ras {

namespace {

constexpr int8_t kFar = 127;

__global__ void k_lev_init(int64_t n, const int32_t* __restrict__ owner, int32_t p, int8_t* lev) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    lev[g] = owner[g] == p ? 0 : kFar;
}

// round l: neighbours of level-l rows (inside the rank's CSR window) get level l + 1
__global__ void k_lev_round(int64_t rb, int64_t nrw, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            int8_t* lev, int l) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrw; r += (int64_t)gridDim.x * blockDim.x) {
    if (lev[rb + r] != l) continue;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int32_t c = col[k];
      if (lev[c] > l + 1) lev[c] = (int8_t)(l + 1);
    }
  }
}

// a row of Omega_p (level <= gamma) outside the window: its row of A is unknown
__global__ void k_lev_check(int64_t n, int64_t rb, int64_t nrw, const int8_t* __restrict__ lev, int gamma, int* bad) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x)
    if (lev[g] <= gamma && (g < rb || g >= rb + nrw)) atomicMin(bad, (int)g);
}

struct LevIn {  // selection predicates over gids
  const int8_t* lev;
  int lo, hi;
  __device__ bool operator()(int32_t g) const { return lev[g] >= lo && lev[g] <= hi; }
};

struct OwnedOf {
  const int32_t* owner;
  int32_t p;
  __device__ int32_t operator()(int32_t g) const { return owner[g] == p ? 1 : 0; }
};

// owned rows of Omega_p get consecutive slots (ascending gid), from off
__global__ void k_own_slots(int64_t m, const int32_t* __restrict__ omega, const int32_t* __restrict__ owner, int32_t p,
                            const int32_t* __restrict__ pre, int64_t off, int32_t* slot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = omega[i];
    if (owner[g] == p) slot[g] = (int32_t)(off + pre[i]);
  }
}

// need_p = (Omega_p \ S_p) u Gamma_p: receive counts per owner subdomain, halo marks
__global__ void k_need(int64_t m, const int32_t* __restrict__ rows, const int32_t* __restrict__ owner, int32_t p,
                       const int32_t* __restrict__ s2r, int32_t me, unsigned long long* cnt, uint8_t* hmark) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = rows[i];
    const int32_t q = owner[g];
    if (q == p) continue;
    atomicAdd(&cnt[q], 1ull);
    if (s2r[q] != me) hmark[g] = 1;
  }
}

struct HaloOfRank {
  const uint8_t* hmark;
  const int32_t* owner;
  const int32_t* s2r;
  int32_t r;
  __device__ bool operator()(int32_t g) const { return hmark[g] && s2r[owner[g]] == r; }
};

__global__ void k_halo_slots(int64_t m, const int32_t* __restrict__ halo, int64_t off, int32_t* slot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    slot[halo[i]] = (int32_t)(off + i);
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// RAII device scratch for the setup (freed before the solver's own buffers are made)
struct Scratch {
  std::vector<void*> p;
  template <class T>
  T* get(size_t n) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    p.push_back(q);
    return (T*)q;
  }
  ~Scratch() {
    for (void* q : p) cudaFree(q);
  }
};

struct HookCtx {
  ras_ctx* c;
  cudaStream_t s;
};

#define DEV_TRY(expr)                                                                \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      set_tls_error(std::string("device setup: ") + #expr + ": " + cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? RAS_ENOMEM : RAS_ECUDA;               \
    }                                                                                \
  } while (0)
#define DEV_ALLOC(ptr) \
  if (!(ptr)) return set_tls_error("device setup: allocation failed"), RAS_ENOMEM

ras_status device_phase1(void* user, ras_plan* pl, const ras_partition* part) {
  HookCtx* H = (HookCtx*)user;
  cudaStream_t s = H->s;
  const int64_t n = pl->n, rb = pl->row_begin, nrw = pl->nrows_win;
  const int32_t P = pl->P, gamma = pl->gamma;
  if (gamma > 120) return set_tls_error("device setup: overlap > 120 (int8 levels)"), RAS_EINVAL;
  Scratch S;
  int32_t* d_owner = S.get<int32_t>(n);
  int64_t* d_rp = S.get<int64_t>(nrw + 1);
  const int64_t nnz = pl->A_ptr[nrw];
  int32_t* d_col = S.get<int32_t>(nnz);
  int8_t* d_lev = S.get<int8_t>(n);
  int32_t* d_s2r = S.get<int32_t>(P);
  int32_t* d_slot = S.get<int32_t>(n);
  uint8_t* d_hmark = S.get<uint8_t>(n);
  unsigned long long* d_cnt = S.get<unsigned long long>(P);
  int32_t* d_sel = S.get<int32_t>(n);     // compaction output
  int32_t* d_sel2 = S.get<int32_t>(n);
  int32_t* d_pre = S.get<int32_t>(n);
  int32_t* d_nsel = S.get<int32_t>(1);
  int* d_bad = S.get<int>(1);
  DEV_ALLOC(d_owner && d_rp && d_col && d_lev && d_s2r && d_slot && d_hmark && d_cnt && d_sel && d_sel2 && d_pre &&
            d_nsel && d_bad);
  DEV_TRY(cudaMemcpyAsync(d_owner, part->owner, n * 4, cudaMemcpyHostToDevice, s));
  DEV_TRY(cudaMemcpyAsync(d_rp, pl->A_ptr, (nrw + 1) * 8, cudaMemcpyHostToDevice, s));
  DEV_TRY(cudaMemcpyAsync(d_col, pl->A_col, std::max<int64_t>(nnz, 1) * 4, cudaMemcpyHostToDevice, s));
  DEV_TRY(cudaMemcpyAsync(d_s2r, pl->sub_to_rank.data(), P * 4, cudaMemcpyHostToDevice, s));
  DEV_TRY(cudaMemsetAsync(d_slot, 0xff, n * 4, s));
  DEV_TRY(cudaMemsetAsync(d_hmark, 0, n, s));
  // CUB temporary storage, sized for the largest call
  cub::CountingInputIterator<int32_t> gids(0);
  size_t tmp_bytes = 0, t1 = 0, t2 = 0;
  cub::DeviceSelect::If(nullptr, t1, gids, d_sel, d_nsel, (int)n, LevIn{d_lev, 0, 0}, s);
  cub::TransformInputIterator<int32_t, OwnedOf, const int32_t*> own_it(d_sel, OwnedOf{d_owner, 0});
  cub::DeviceScan::ExclusiveSum(nullptr, t2, own_it, d_pre, (int)n, s);
  tmp_bytes = std::max(t1, t2);
  void* d_tmp = S.get<char>(tmp_bytes);
  DEV_ALLOC(d_tmp);
  auto select = [&](auto pred, int32_t* out, int64_t* count) -> ras_status {
    size_t tb = tmp_bytes;
    DEV_TRY(cub::DeviceSelect::If(d_tmp, tb, gids, out, d_nsel, (int)n, pred, s));
    int32_t h = 0;
    DEV_TRY(cudaMemcpyAsync(&h, d_nsel, 4, cudaMemcpyDeviceToHost, s));
    DEV_TRY(cudaStreamSynchronize(s));
    *count = h;
    return RAS_OK;
  };
  const int32_t nl = (int32_t)pl->subs.size();
  int64_t off = 0;
  std::vector<unsigned long long> cnt(P);
  std::vector<int32_t> buf;
  for (int32_t lp = 0; lp < nl; ++lp) {
    auto& SP = pl->subs[lp];
    const int32_t p = SP.p;
    // ---- gamma-hop levels (R1) ----
    k_lev_init<<<grid_for(n), 256, 0, s>>>(n, d_owner, p, d_lev);
    for (int l = 0; l <= gamma; ++l) k_lev_round<<<grid_for(nrw), 256, 0, s>>>(rb, nrw, d_rp, d_col, d_lev, l);
    int bad = INT32_MAX;
    DEV_TRY(cudaMemcpyAsync(d_bad, &bad, 4, cudaMemcpyHostToDevice, s));
    k_lev_check<<<grid_for(n), 256, 0, s>>>(n, rb, nrw, d_lev, gamma, d_bad);
    DEV_TRY(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
    DEV_TRY(cudaStreamSynchronize(s));
    if (bad != INT32_MAX)
      return set_tls_error("row " + std::to_string(bad) + " of an Omega_p is outside the CSR row window [" +
                           std::to_string(rb) + ", " + std::to_string(rb + nrw) + ")"),
             RAS_EINVAL;
    // ---- Omega_p (levels <= gamma) and Gamma_p (level gamma + 1), ascending ----
    int64_t nom = 0, ngh = 0;
    TRY(select(LevIn{d_lev, 0, gamma}, d_sel, &nom));
    TRY(select(LevIn{d_lev, gamma + 1, gamma + 1}, d_sel2, &ngh));
    buf.resize(std::max(nom, ngh));
    DEV_TRY(cudaMemcpyAsync(buf.data(), d_sel, nom * 4, cudaMemcpyDeviceToHost, s));
    DEV_TRY(cudaStreamSynchronize(s));
    SP.omega.assign(buf.begin(), buf.begin() + nom);
    DEV_TRY(cudaMemcpyAsync(buf.data(), d_sel2, ngh * 4, cudaMemcpyDeviceToHost, s));
    DEV_TRY(cudaStreamSynchronize(s));
    SP.ghosts.assign(buf.begin(), buf.begin() + ngh);
    SP.owned.resize(nom);
    for (int64_t i = 0; i < nom; ++i) SP.owned[i] = part->owner[SP.omega[i]] == p;
    // ---- owned slots: consecutive over S_p ascending ----
    {
      cub::TransformInputIterator<int32_t, OwnedOf, const int32_t*> it(d_sel, OwnedOf{d_owner, p});
      size_t tb = tmp_bytes;
      DEV_TRY(cub::DeviceScan::ExclusiveSum(d_tmp, tb, it, d_pre, (int)nom, s));
      k_own_slots<<<grid_for(nom), 256, 0, s>>>(nom, d_sel, d_owner, p, d_pre, off, d_slot);
    }
    SP.own_off = off;
    SP.nown = 0;
    for (int64_t i = 0; i < nom; ++i)
      if (SP.owned[i]) {
        pl->own_gid.push_back(SP.omega[i]);
        ++SP.nown;
      }
    off += SP.nown;
    // ---- need_p: receive counts per owner subdomain (Fig. 2) and halo marks ----
    DEV_TRY(cudaMemsetAsync(d_cnt, 0, P * 8, s));
    k_need<<<grid_for(nom), 256, 0, s>>>(nom, d_sel, d_owner, p, d_s2r, pl->rank, d_cnt, d_hmark);
    k_need<<<grid_for(ngh), 256, 0, s>>>(ngh, d_sel2, d_owner, p, d_s2r, pl->rank, d_cnt, d_hmark);
    DEV_TRY(cudaMemcpyAsync(cnt.data(), d_cnt, P * 8, cudaMemcpyDeviceToHost, s));
    DEV_TRY(cudaStreamSynchronize(s));
    for (int32_t q = 0; q < P; ++q)
      if (cnt[q]) {
        SP.nbr_subs.push_back(q);
        SP.nbr_cnt.push_back((int64_t)cnt[q]);
      }
  }
  pl->n_own = off;
  // ---- halo: sorted by (owning rank, gid); slots after the owned ones ----
  pl->halo_off.assign(pl->world + 1, 0);
  pl->halo_gid.clear();
  for (int32_t r = 0; r < pl->world; ++r) {
    int64_t m = 0;
    TRY(select(HaloOfRank{d_hmark, d_owner, d_s2r, r}, d_sel, &m));
    if (m) {
      k_halo_slots<<<grid_for(m), 256, 0, s>>>(m, d_sel, pl->n_own + (int64_t)pl->halo_gid.size(), d_slot);
      buf.resize(m);
      DEV_TRY(cudaMemcpyAsync(buf.data(), d_sel, m * 4, cudaMemcpyDeviceToHost, s));
      DEV_TRY(cudaStreamSynchronize(s));
      pl->halo_gid.insert(pl->halo_gid.end(), buf.begin(), buf.begin() + m);
    }
    pl->halo_off[r + 1] = (int64_t)pl->halo_gid.size();
  }
  pl->n_halo = (int64_t)pl->halo_gid.size();
  pl->slot.resize(n);
  DEV_TRY(cudaMemcpyAsync(pl->slot.data(), d_slot, n * 4, cudaMemcpyDeviceToHost, s));
  DEV_TRY(cudaStreamSynchronize(s));
  DEV_TRY(cudaGetLastError());
  return RAS_OK;
}

}  // namespace

ras_status plan_build_device(ras_ctx* c, ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part,
                             int32_t overlap) {
  HookCtx H{c, c->stream};
  PlanDeviceHook hook{device_phase1, &H};
  return plan_build_ex(out, A, b, part, overlap, c->rank, c->world, &hook);
}

}  // namespace ras
