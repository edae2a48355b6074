// sm_100a kernels of one RAS sweep (scope rows a1-a5).  FP64, no tensor cores:
// every kernel here is an HBM-streaming sparse/vector kernel.
//
// Layout (see include/ras_plan.h): the rank's subdomains' Omega_p rows are
// concatenated into one padded "row space"; matrices are SELL-32 (slice = 32
// consecutive rows stored column-major, so lane i of a warp reads entry k of
// row i at base + 32k + i: one coalesced 256 B value load + 128 B index load
// per k).  A CTA (256 threads) processes one TILE of kRPT*256 rows that never
// straddles subdomains; every thread owns kRPT rows (row0 + j*256 + tid) and
// issues all their loads before using any (memory-level parallelism).
// Per-subdomain dot products are reduced deterministically: every CTA writes
// its partial, the last CTA of the subdomain (atomic ticket) sums the partials
// in fixed order and applies the PCG scalar update.
#pragma once

#include <cstdint>

namespace ras {

constexpr int kThreads = 256;
constexpr int kRPT = 4;                     // rows per thread
constexpr int kTileRows = kThreads * kRPT;  // rows per CTA tile (plan tile_rows)
constexpr int kNP = 4;                      // partial slots per tile
constexpr int kMaxW = 8;                    // unrolled SELL width (wider slices take the loop path)

struct Tiles {
  const int4* tile;               // {row0, nrows, local subdomain, 0}
  const int64_t* sub_tile_begin;  // per local subdomain
  const int32_t* sub_ntiles;
};

struct Sell {
  const int64_t* sptr;
  const int32_t* col;
  const double* val;
};

// Per local subdomain scalars (struct of arrays, one allocation each).
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

// Stop control: sync = one global word (per_sub = 0); async = one word per
// local subdomain (per_sub = 1).
struct Ctl {
  const volatile int32_t* stop;
  int32_t per_sub;
};

__device__ __forceinline__ bool stopped(const Ctl& C, int lp) {
  return C.stop && C.stop[C.per_sub ? lp : 0];
}

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

// Sum_k val[e_k] * x[col[e_k]] over SELL-32 row `row` (entries in ascending
// column order as stored).  Matrix data is streamed with evict-first loads so
// the gathered vector keeps its L2 lines.
__device__ __forceinline__ double sell_dot(const Sell& M, int64_t row, const double* __restrict__ x) {
  const int64_t s = row >> 5;
  const int lane = (int)(row & 31);
  const int64_t base = __ldg(&M.sptr[s]);
  const int w = (int)((__ldg(&M.sptr[s + 1]) - base) >> 5);
  const double* vp = M.val + base + lane;
  const int32_t* cp = M.col + base + lane;
  double acc = 0.0;
  if (w <= kMaxW) {
    double v[kMaxW];
    int32_t c[kMaxW];
#pragma unroll
    for (int k = 0; k < kMaxW; ++k)
      if (k < w) {
        v[k] = __ldcs(vp + 32 * k);
        c[k] = __ldcs(cp + 32 * k);
      }
#pragma unroll
    for (int k = 0; k < kMaxW; ++k)
      if (k < w) acc += v[k] * __ldg(&x[c[k]]);
  } else {
    for (int k = 0; k < w; ++k) acc += __ldcs(vp + 32 * k) * __ldg(&x[__ldcs(cp + 32 * k)]);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// a1+a2: restrict + residual + PCG start.
//   r = b~ - [A_p|B_p] x (x read in place from owned/halo storage: restrict),
//   JAC: z = D^-1 r, p = z; partials: rho = r.z, ||r~||^2, owned ||r~||^2.
//   !JAC (IC(0)/ILU(0)): only r and the norms; z = M^-1 r follows (trsv).
// ---------------------------------------------------------------------------
template <bool JAC = true>
static __global__ void __launch_bounds__(kThreads) k_residual(int64_t tile_base, Tiles T, Sell R,
                                                              const double* __restrict__ b,
                                                              const double* __restrict__ diag,
                                                              const int32_t* __restrict__ own_slot,
                                                              const double* __restrict__ x, double* __restrict__ r,
                                                              double* __restrict__ p, Scal S, Ctl C) {
  __shared__ double sh[3][kThreads / 32];
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp)) return;
  double v[3] = {0.0, 0.0, 0.0};
  double bi[kRPT], di[kRPT], ax[kRPT];
  int32_t os[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      bi[j] = __ldcs(&b[row]);
      di[j] = __ldcs(&diag[row]);
      os[j] = __ldcs(&own_slot[row]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) ax[j] = sell_dot(R, ti.x + lr, x);
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      const double ri = bi[j] - ax[j];
      r[row] = ri;
      if (JAC) {
        const double zi = __drcp_rn(di[j]) * ri;
        p[row] = zi;
        v[0] += ri * zi;
      }
      v[1] += ri * ri;
      v[2] += os[j] >= 0 ? ri * ri : 0.0;
    }
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
      // "if rho == 0: break" (R7); IC path: decided after z = M^-1 r (k_zdot<true>)
      S.active[lp] = JAC ? (o[0] != 0.0) : 1;
      S.its[lp] = 0;
      S.ticket[lp] = 0u;
    }
  }
}

// a3 pass 1: q = A_p p (diag + SELL off-diagonal), sigma = p.q; last CTA: alpha.
static __global__ void __launch_bounds__(kThreads) k_spmv_dot(int64_t tile_base, Tiles T, Sell L,
                                                              const double* __restrict__ diag,
                                                              const double* __restrict__ p, double* __restrict__ q,
                                                              Scal S, Ctl C) {
  __shared__ double sh[1][kThreads / 32];
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  double v[1] = {0.0};
  double pi[kRPT], di[kRPT], ax[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      pi[j] = __ldg(&p[row]);
      di[j] = __ldcs(&diag[row]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) ax[j] = sell_dot(L, ti.x + lr, p);
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const double qi = di[j] * pi[j] + ax[j];
      q[ti.x + lr] = qi;
      v[0] += pi[j] * qi;
    }
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
// JAC: z = D^-1 r; partials r.z, r.r; last CTA: inner stop test, beta, rho.
// !JAC: only r.r (inner stop test, iteration cap); rho' after the trisolves.
template <bool JAC = true>
static __global__ void __launch_bounds__(kThreads) k_update_dot(int64_t tile_base, Tiles T,
                                                                const double* __restrict__ diag,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ q, double* __restrict__ r,
                                                                double* __restrict__ d, Scal S, Ctl C, int32_t m,
                                                                double inner_tol) {
  __shared__ double sh[2][kThreads / 32];
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double alpha = S.alpha[lp];
  const bool first = S.its[lp] == 1;
  double v[2] = {0.0, 0.0};
  double pi[kRPT], qi[kRPT], ri[kRPT], di[kRPT], gi[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      pi[j] = __ldcs(&p[row]);
      qi[j] = __ldcs(&q[row]);
      ri[j] = __ldcs(&r[row]);
      if (JAC) gi[j] = __ldcs(&diag[row]);
      di[j] = first ? 0.0 : __ldcs(&d[row]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      const double dn = first ? alpha * pi[j] : di[j] + alpha * pi[j];
      const double rn = ri[j] - alpha * qi[j];
      d[row] = dn;
      r[row] = rn;
      if (JAC) {
        const double zi = __drcp_rn(gi[j]) * rn;
        v[0] += rn * zi;
      }
      v[1] += rn * rn;
    }
  }
  block_sum<2>(v, sh);
  if (tile_partials_last<2>(v, t, lp, T, S)) {
    double o[2];
    reduce_sub_partials<2>(o, lp, T, S, sh);
    if (threadIdx.x == 0) {
      S.rr[lp] = o[1];
      if (inner_tol > 0.0 && sqrt(o[1]) <= inner_tol * sqrt(S.rt2[lp])) {
        S.active[lp] = 0;  // inner tolerance reached (exact mode / eta)
      } else if (!JAC) {
        if (S.its[lp] >= m) S.active[lp] = 0;  // z, rho', p of the last iteration are never used
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
static __global__ void __launch_bounds__(kThreads) k_pupdate(int64_t tile_base, Tiles T,
                                                             const double* __restrict__ diag,
                                                             const double* __restrict__ r, double* __restrict__ p,
                                                             Scal S, Ctl C) {
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double beta = S.beta[lp];
  double gi[kRPT], ri[kRPT], pi[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      gi[j] = __ldcs(&diag[row]);
      ri[j] = __ldcs(&r[row]);
      pi[j] = __ldcs(&p[row]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) p[ti.x + lr] = __drcp_rn(gi[j]) * ri[j] + beta * pi[j];
  }
}

// ---------------------------------------------------------------------------
// a3' (IC(0)/ILU(0)-PCG): M = L U, z = U^-1 L^-1 r by two level-scheduled
// triangular solves (P320-323, level-set strategy).
// ---------------------------------------------------------------------------
struct TriDev {
  const int32_t* rows;    // level-ordered row-space rows
  const int32_t* rp;      // entry offsets per level-ordered position
  const int32_t* col;     // dependency rows
  const double* val;
  const double* diag;     // divisor per row-space row
  const int4* chunk;      // {rows begin, rows end, local subdomain, level}
  const int32_t* batched; // chunk order of a batched (all-subdomain) solve
  const int32_t* sub_lev_off;
  const int32_t* lev_nchunks;
};

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// out[i] = (in[i] - sum_j T_ij out[j]) / diag[i], rows in level order.
// Chunks (256 rows of one level of one subdomain) are claimed from an atomic
// counter in level order; a chunk of level l of subdomain p first waits until
// every chunk of level l-1 of p has completed.  A waited-on chunk was claimed
// earlier by a running CTA, so the wait always terminates (no co-residency
// assumption, no inter-launch waiting).
static __global__ void __launch_bounds__(kThreads) k_trsv(TriDev T, int use_batched, int32_t c0, int32_t nchunk,
                                                          uint32_t* counter, int32_t* lev_done,
                                                          const double* __restrict__ in, double* out,
                                                          const int32_t* __restrict__ active, Ctl C) {
  __shared__ int s_c;
  for (;;) {
    if (threadIdx.x == 0) s_c = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int c = s_c;
    __syncthreads();
    if (c >= nchunk) return;
    const int cid = use_batched ? T.batched[c] : c0 + c;
    const int4 ch = T.chunk[cid];
    const int lp = ch.z, lev = ch.w;
    const int32_t* done = lev_done + T.sub_lev_off[lp];
    const bool skip = stopped(C, lp) || !active[lp];
    if (!skip && lev > 0 && threadIdx.x == 0) {
      const int32_t need = T.lev_nchunks[T.sub_lev_off[lp] + lev - 1];
      while (ld_acquire_gpu(done + lev - 1) < need) __nanosleep(64);
    }
    __syncthreads();
    const int k = ch.x + threadIdx.x;
    if (!skip && k < ch.y) {
      const int32_t i = __ldg(&T.rows[k]);
      double s = __ldg(&in[i]);
      const int32_t e1 = __ldg(&T.rp[k + 1]);
      for (int32_t e = __ldg(&T.rp[k]); e < e1; ++e) s -= __ldg(&T.val[e]) * __ldcg(&out[__ldg(&T.col[e])]);
      __stcg(&out[i], s / __ldg(&T.diag[i]));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&lev_done[T.sub_lev_off[lp] + lev], 1);
    }
  }
}

// IC path, after z = M^-1 r.  INIT (PCG start): p = z, rho = r.z, active = rho != 0.
// !INIT: rho' = r.z, beta = rho'/rho, rho = rho' (rho' == 0 -> stop, R7).
template <bool INIT>
static __global__ void __launch_bounds__(kThreads) k_zdot(int64_t tile_base, Tiles T, const double* __restrict__ r,
                                                          const double* __restrict__ z, double* __restrict__ p, Scal S,
                                                          Ctl C) {
  __shared__ double sh[1][kThreads / 32];
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  double v[1] = {0.0};
  double ri[kRPT], zi[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      ri[j] = __ldcs(&r[ti.x + lr]);
      zi[j] = __ldcs(&z[ti.x + lr]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      v[0] += ri[j] * zi[j];
      if (INIT) p[ti.x + lr] = zi[j];
    }
  }
  block_sum<1>(v, sh);
  if (tile_partials_last<1>(v, t, lp, T, S)) {
    double o[1];
    reduce_sub_partials<1>(o, lp, T, S, sh);
    if (threadIdx.x == 0) {
      if (INIT) {
        S.rho[lp] = o[0];
        S.active[lp] = o[0] != 0.0;
      } else {
        S.beta[lp] = o[0] / S.rho[lp];
        S.rho[lp] = o[0];
        if (o[0] == 0.0) S.active[lp] = 0;
      }
      S.ticket[lp] = 0u;
    }
  }
}

// IC path: p = z + beta p.
static __global__ void __launch_bounds__(kThreads) k_pupdate_z(int64_t tile_base, Tiles T,
                                                               const double* __restrict__ z, double* __restrict__ p,
                                                               Scal S, Ctl C) {
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double beta = S.beta[lp];
  double zi[kRPT], pi[kRPT];
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      zi[j] = __ldcs(&z[ti.x + lr]);
      pi[j] = __ldcs(&p[ti.x + lr]);
    }
  }
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) p[ti.x + lr] = zi[j] + beta * pi[j];
  }
}

// a4: restricted prolongation x[S_p] += d[S_p] (overlap part of d discarded).
static __global__ void __launch_bounds__(kThreads) k_prolong(int64_t tile_base, Tiles T,
                                                             const int32_t* __restrict__ own_slot,
                                                             const double* __restrict__ d, double* __restrict__ x,
                                                             Scal S, Ctl C) {
  const int64_t t = tile_base + blockIdx.x;
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || S.its[lp] == 0) return;  // no PCG step taken: d == 0
#pragma unroll
  for (int j = 0; j < kRPT; ++j) {
    const int lr = j * kThreads + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      const int32_t s = __ldcs(&own_slot[row]);
      if (s >= 0) x[s] = x[s] + __ldcs(&d[row]);
    }
  }
}

// a5 (sync): pack owned values for the NCCL sends.
static __global__ void k_pack(int64_t count, const int32_t* __restrict__ slots, const double* __restrict__ x,
                              double* __restrict__ out, Ctl C) {
  if (stopped(C, 0)) return;
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

static __global__ void k_sync_check(const double* __restrict__ r2_global, double b2_global, double tol,
                                    int64_t max_iters, SyncState* st, int32_t* stop_flag,
                                    volatile int32_t* host_stop) {
  if (threadIdx.x || blockIdx.x) return;
  if (!st->stop) {
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
  }
  if (host_stop) *host_stop = st->stop;  // mapped pinned ring slot of this sweep
}

static __global__ void k_count_active(int nl, const int32_t* __restrict__ active, int32_t* out) {
  if (threadIdx.x || blockIdx.x) return;
  int c = 0;
  for (int i = 0; i < nl; ++i) c += active[i] != 0;
  *out = c;
}

// x0 (global order, device copy of the caller's host buffer) -> storage order
static __global__ void k_scatter_x0(int64_t n_own, int64_t n_halo, const int32_t* __restrict__ own_gid,
                                    const int32_t* __restrict__ halo_gid, const double* __restrict__ xg,
                                    double* __restrict__ x) {
  const int64_t tot = n_own + n_halo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = i < n_own ? xg[own_gid[i]] : xg[halo_gid[i - n_own]];
}

// owned storage -> global order (x_out gather, P242)
static __global__ void k_gather_x(int64_t n_own, const int32_t* __restrict__ own_gid, const double* __restrict__ x,
                                  double* __restrict__ xg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_own; i += (int64_t)gridDim.x * blockDim.x)
    xg[own_gid[i]] = x[i];
}

}  // namespace ras
