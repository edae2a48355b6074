// sm_100a kernels of one RAS sweep (scope rows a1-a5).  FP64, no tensor cores:
// every kernel here is an HBM-streaming sparse/vector kernel.
//
// Layout (see include/ras_plan.h): the rank's subdomains' Omega_p rows are
// concatenated into one padded "row space"; matrices are SELL-32 (slice = 32
// consecutive rows stored column-major, so lane i of a warp reads entry k of
// row i at base + 32k + i: one coalesced 256 B value load + 128 B index load
// per k).  A CTA processes one TILE of rows that never straddles subdomains;
// per-subdomain dot products are reduced deterministically: every CTA writes
// its partial, the last CTA of the subdomain (atomic ticket) sums the partials
// in fixed order and applies the PCG scalar update.
#pragma once

#include <cstdint>

namespace ras {

constexpr int kThreads = 256;  // = TILE rows: one 32-row slice per warp
constexpr int kNP = 4;         // partial slots per tile

struct Tiles {
  const int32_t* tile_sub;
  const int64_t* tile_row0;
  const int32_t* tile_nrows;
  const int64_t* sub_tile_begin;  // per local subdomain
  const int32_t* sub_ntiles;
};

struct Sell {
  const int64_t* sptr;
  const int32_t* col;
  const double* val;
};

// Per local subdomain scalars (struct of arrays, one allocation).
struct Scal {
  double* rt2;     // ||r~_p||^2 over Omega_p (Eq. 2 numerator, inner stop)
  double* rho;     // r.z
  double* own2;    // sum over owned rows of r~^2 (global criterion partial)
  double* alpha;
  double* beta;
  double* rr;      // ||r||^2 of the current inner residual
  int32_t* active; // PCG still iterating
  int32_t* its;    // PCG iterations performed this sweep
  uint32_t* ticket;
  int64_t* inner_total;  // PCG iterations accumulated over the solve
  double* partials;  // ntiles * kNP
};

struct Ctl {
  volatile int32_t* stop;  // sync: global stop flag (device); nullptr in async
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum of NV values; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*sh)[kThreads / 32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double s = warp_sum(v[j]);
    if (lane == 0) sh[j][w] = s;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = lane < kThreads / 32 ? sh[j][lane] : 0.0;
      s = warp_sum(s);
      v[j] = s;
    }
  }
  __syncthreads();
}

// Writes this tile's partials; returns true in every thread of the CTA that
// is the last one of subdomain lp to finish (that CTA then owns the reduction).
template <int NV>
__device__ __forceinline__ bool tile_partials_last(const double (&v)[NV], int64_t t, int lp, const Tiles& T,
                                                   const Scal& S) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) S.partials[t * kNP + j] = v[j];
    __threadfence();
    const uint32_t prev = atomicAdd(&S.ticket[lp], 1u);
    s_last = (prev == (uint32_t)T.sub_ntiles[lp] - 1u);
  }
  __syncthreads();
  return s_last != 0;
}

// In the last CTA: fixed-order sum of subdomain lp's partials (result in thread 0).
template <int NV>
__device__ __forceinline__ void reduce_sub_partials(double (&out)[NV], int lp, const Tiles& T, const Scal& S,
                                                    double (*sh)[kThreads / 32]) {
  __threadfence();
  const int64_t tb = T.sub_tile_begin[lp];
  const int nt = T.sub_ntiles[lp];
#pragma unroll
  for (int j = 0; j < NV; ++j) out[j] = 0.0;
  for (int i = threadIdx.x; i < nt; i += kThreads) {
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] += __ldcg(&S.partials[(tb + i) * kNP + j]);
  }
  block_sum<NV>(out, sh);
}

__device__ __forceinline__ double sell_dot(const Sell& M, int64_t row, const double* __restrict__ x) {
  const int64_t s = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t base = M.sptr[s];
  const int w = (int)((M.sptr[s + 1] - base) >> 5);
  double acc = 0.0;
  for (int k = 0; k < w; ++k) {
    const int64_t e = base + (int64_t)k * 32 + lane;
    acc += __ldg(&M.val[e]) * __ldg(&x[__ldg(&M.col[e])]);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// a1+a2: restrict + residual + PCG start.
//   r = b~ - [A_p|B_p] x (x read in place from owned/halo storage: restrict),
//   z = D^-1 r, p = z; partials: rho = r.z, ||r~||^2, owned ||r~||^2.
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(kThreads) k_residual(int64_t tile_base, Tiles T, Sell R, const double* __restrict__ b,
                                                       const double* __restrict__ diag,
                                                       const int32_t* __restrict__ own_slot,
                                                       const double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ p, Scal S, Ctl C) {
  __shared__ double sh[3][kThreads / 32];
  if (C.stop && *C.stop) return;
  const int64_t t = tile_base + blockIdx.x;
  const int lp = T.tile_sub[t];
  const int64_t row = T.tile_row0[t] + threadIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  if ((int)threadIdx.x < T.tile_nrows[t]) {
    const double ri = __ldg(&b[row]) - sell_dot(R, row, x);
    const double zi = __drcp_rn(__ldg(&diag[row])) * ri;
    r[row] = ri;
    p[row] = zi;
    v[0] = ri * zi;
    v[1] = ri * ri;
    v[2] = __ldg(&own_slot[row]) >= 0 ? ri * ri : 0.0;
  }
  block_sum<3>(v, sh);
  if (tile_partials_last<3>(v, t, lp, T, S)) {
    double o[3];
    reduce_sub_partials<3>(o, lp, T, S, sh);
    if (threadIdx.x == 0) {
      S.rho[lp] = o[0];
      S.rt2[lp] = o[1];
      S.own2[lp] = o[2];
      S.rr[lp] = o[1];
      S.active[lp] = (o[0] != 0.0);  // "if rho == 0: break" (R7)
      S.its[lp] = 0;
      S.ticket[lp] = 0u;
    }
  }
}

// a3 pass 1: q = A_p p (diag + SELL off-diagonal), sigma = p.q; last CTA: alpha.
static __global__ void __launch_bounds__(kThreads) k_spmv_dot(int64_t tile_base, Tiles T, Sell L,
                                                       const double* __restrict__ diag, const double* __restrict__ p,
                                                       double* __restrict__ q, Scal S, Ctl C) {
  __shared__ double sh[1][kThreads / 32];
  if (C.stop && *C.stop) return;
  const int64_t t = tile_base + blockIdx.x;
  const int lp = T.tile_sub[t];
  if (!S.active[lp]) return;
  const int64_t row = T.tile_row0[t] + threadIdx.x;
  double v[1] = {0.0};
  if ((int)threadIdx.x < T.tile_nrows[t]) {
    const double pi = __ldg(&p[row]);
    const double qi = __ldg(&diag[row]) * pi + sell_dot(L, row, p);
    q[row] = qi;
    v[0] = pi * qi;
  }
  block_sum<1>(v, sh);
  if (tile_partials_last<1>(v, t, lp, T, S)) {
    double o[1];
    reduce_sub_partials<1>(o, lp, T, S, sh);
    if (threadIdx.x == 0) {
      const double sigma = o[0];
      if (sigma == 0.0) {  // "if sigma == 0: break" (R7)
        S.active[lp] = 0;
        S.alpha[lp] = 0.0;
      } else {
        S.alpha[lp] = S.rho[lp] / sigma;
        S.its[lp] += 1;
        S.inner_total[lp] += 1;
      }
      S.ticket[lp] = 0u;
    }
  }
}

// a3 pass 2: d += alpha p (d = alpha p on the first iteration), r -= alpha q,
// z = D^-1 r; partials r.z, r.r; last CTA: inner stop test, beta, rho.
static __global__ void __launch_bounds__(kThreads) k_update_dot(int64_t tile_base, Tiles T, const double* __restrict__ diag,
                                                         const double* __restrict__ p, const double* __restrict__ q,
                                                         double* __restrict__ r, double* __restrict__ d, Scal S,
                                                         Ctl C, int32_t m, double inner_tol) {
  __shared__ double sh[2][kThreads / 32];
  if (C.stop && *C.stop) return;
  const int64_t t = tile_base + blockIdx.x;
  const int lp = T.tile_sub[t];
  if (!S.active[lp]) return;
  const double alpha = S.alpha[lp];
  const bool first = S.its[lp] == 1;
  const int64_t row = T.tile_row0[t] + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if ((int)threadIdx.x < T.tile_nrows[t]) {
    const double pi = __ldg(&p[row]);
    const double di = first ? alpha * pi : d[row] + alpha * pi;
    const double ri = r[row] - alpha * __ldg(&q[row]);
    d[row] = di;
    r[row] = ri;
    const double zi = __drcp_rn(__ldg(&diag[row])) * ri;
    v[0] = ri * zi;
    v[1] = ri * ri;
  }
  block_sum<2>(v, sh);
  if (tile_partials_last<2>(v, t, lp, T, S)) {
    double o[2];
    reduce_sub_partials<2>(o, lp, T, S, sh);
    if (threadIdx.x == 0) {
      S.rr[lp] = o[1];
      if (inner_tol > 0.0 && sqrt(o[1]) <= inner_tol * sqrt(S.rt2[lp])) {
        S.active[lp] = 0;  // inner tolerance reached (exact mode / eta)
      } else {
        const double rho_new = o[0];
        S.beta[lp] = rho_new / S.rho[lp];
        S.rho[lp] = rho_new;
        if (S.its[lp] >= m || rho_new == 0.0) S.active[lp] = 0;
      }
      S.ticket[lp] = 0u;
    }
  }
}

// a3 pass 3: p = D^-1 r + beta p.
static __global__ void __launch_bounds__(kThreads) k_pupdate(int64_t tile_base, Tiles T, const double* __restrict__ diag,
                                                      const double* __restrict__ r, double* __restrict__ p, Scal S,
                                                      Ctl C) {
  if (C.stop && *C.stop) return;
  const int64_t t = tile_base + blockIdx.x;
  const int lp = T.tile_sub[t];
  if (!S.active[lp]) return;
  const double beta = S.beta[lp];
  const int64_t row = T.tile_row0[t] + threadIdx.x;
  if ((int)threadIdx.x < T.tile_nrows[t]) {
    const double zi = __drcp_rn(__ldg(&diag[row])) * __ldg(&r[row]);
    p[row] = zi + beta * p[row];
  }
}

// a4: restricted prolongation x[S_p] += d[S_p] (overlap part of d discarded).
static __global__ void __launch_bounds__(kThreads) k_prolong(int64_t tile_base, Tiles T, const int32_t* __restrict__ own_slot,
                                                      const double* __restrict__ d, double* __restrict__ x, Scal S,
                                                      Ctl C) {
  if (C.stop && *C.stop) return;
  const int64_t t = tile_base + blockIdx.x;
  const int lp = T.tile_sub[t];
  if (S.its[lp] == 0) return;  // no PCG step taken: d == 0
  const int64_t row = T.tile_row0[t] + threadIdx.x;
  if ((int)threadIdx.x < T.tile_nrows[t]) {
    const int32_t s = __ldg(&own_slot[row]);
    if (s >= 0) x[s] = x[s] + __ldg(&d[row]);
  }
}

// a5 (sync): pack owned values for the NCCL sends.
static __global__ void k_pack(int64_t count, const int32_t* __restrict__ slots, const double* __restrict__ x,
                       double* __restrict__ out, Ctl C) {
  if (C.stop && *C.stop) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[__ldg(&slots[i])];
}

// a6 (sync): sum owned partials over local subdomains in fixed order.
static __global__ void k_sum_own(int nl, const double* __restrict__ own2, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nl; ++i) s += own2[i];
    *out = s;
  }
}

// a6 (sync): global criterion ||b - A x^k|| < tol ||b|| (P344-346, R13).
struct SyncState {
  int32_t stop, converged;
  int64_t sweeps;   // sweeps applied so far (k)
  double rel;       // relative residual of x^k
};

static __global__ void k_sync_check(const double* __restrict__ r2_global, double b2_global, double tol, int64_t max_iters,
                             SyncState* st, int32_t* stop_flag, volatile int32_t* host_stop) {
  if (threadIdx.x || blockIdx.x) return;
  if (st->stop) return;
  const double r2 = *r2_global;
  const double rel = b2_global > 0.0 ? sqrt(r2) / sqrt(b2_global) : (r2 == 0.0 ? 0.0 : INFINITY);
  st->rel = rel;
  const bool conv = b2_global > 0.0 ? (rel < tol) : (r2 == 0.0);
  if (conv) {
    st->stop = 1;
    st->converged = 1;
  } else if (st->sweeps >= max_iters) {
    st->stop = 1;
  } else {
    st->sweeps += 1;
  }
  if (st->stop) *stop_flag = 1;
  if (host_stop) *host_stop = st->stop;  // mapped pinned ring slot of this sweep
}

static __global__ void k_count_active(int nl, const int32_t* __restrict__ active, int32_t* out) {
  if (threadIdx.x || blockIdx.x) return;
  int c = 0;
  for (int i = 0; i < nl; ++i) c += active[i] != 0;
  *out = c;
}

}  // namespace ras
