// sm_100a kernels of one RAS sweep (scope rows a1-a5, a3').  FP64, no tensor
// cores: every kernel here is an HBM-streaming sparse/vector kernel.
//
// Layout (see include/ras_plan.h): the rank's subdomains' Omega_p rows are
// concatenated into one padded "row space"; matrices are SELL-32 (slice = 32
// consecutive rows stored column-major, so lane i of a warp reads entry k of
// row i at base + 32k + i: one coalesced 256 B value load + 128 B index load
// per k).  A CTA processes one TILE of kTileRows rows that never straddles
// subdomains; each kernel has its own CTA size NT (tuned, see below) and every
// thread owns RPT = kTileRows / NT rows (row0 + j*NT + tid), issuing all their
// loads before using any (memory-level parallelism).  Consecutive streaming
// launches walk the tiles in alternating directions (Tiles::rev) so each one
// starts on the vectors the previous one left in the 126 MB L2.
//
// Per-subdomain dot products are reduced deterministically and without
// atomics or fences in the streaming kernels: every CTA writes its partial
// sums slot-major to partials[slot][tile]; a small k_finish kernel (one CTA per
// subdomain) sums them in fixed order and applies the PCG scalar update
// (alpha, beta, stop tests) that the next streaming kernel reads.  Kernels are
// chained with programmatic dependent launch (pdl_start).
#pragma once

#include <cstdint>

namespace ras {

constexpr int kThreads = 256;               // default CTA size (trisolve, finish helpers)
constexpr int kWarps = kThreads / 32;
#ifndef RAS_RPT
#define RAS_RPT 4
#endif
constexpr int kTileRows = 256 * RAS_RPT;    // rows per CTA tile (plan tile_rows)
// Threads per CTA (and the minimum resident CTAs per SM, i.e. the register
// budget) of each streaming kernel; rows per thread = kTileRows / threads.
// Tuned on B200 (round 1 sweep): the gather kernels want more,
// lighter threads (2 rows each), the pure streams 4 rows per thread.
// k_residual on the row-pattern (SELL-Z) matrix: 256 threads x 8 CTAs/SM (4 rows
// per thread, full occupancy) measured 268 us vs 281 us for 512 x 4 on C2
// (profiles/r01_exp_residual_cta.txt); the SELL-32 instantiations keep 512 x 4
// (they spill 2-3x more at 32 registers and were not re-measured).
#ifndef RAS_NT_RES
#define RAS_NT_RES 512
#endif
#ifndef RAS_MB_RES
#define RAS_MB_RES 4
#endif
#ifndef RAS_NT_RES_Z
#define RAS_NT_RES_Z 256
#endif
#ifndef RAS_MB_RES_Z
#define RAS_MB_RES_Z 8
#endif
#ifndef RAS_NT_SPMV
#define RAS_NT_SPMV 512
#endif
#ifndef RAS_MB_SPMV
#define RAS_MB_SPMV 4
#endif
#ifndef RAS_NT_UPD
#define RAS_NT_UPD 512
#endif
#ifndef RAS_MB_UPD
#define RAS_MB_UPD 4
#endif
#ifndef RAS_NT_STREAM
#define RAS_NT_STREAM 256
#endif
#ifndef RAS_MB_STREAM
#define RAS_MB_STREAM 6
#endif
constexpr int kNT_RES = RAS_NT_RES, kNT_RES_Z = RAS_NT_RES_Z, kNT_SPMV = RAS_NT_SPMV, kNT_UPD = RAS_NT_UPD, kNT_STREAM = RAS_NT_STREAM;
constexpr int kNP = 4;                      // partial slots per warp
constexpr int kMaxW = 8;                    // unrolled SELL width (wider slices take the loop path)
constexpr int kStageMax = 4096;             // max p span staged in shared memory by k_spmv_dot (32 KB)

struct Tiles {
  const int4* tile;               // {row0, nrows, local subdomain, 0}
  const int64_t* sub_tile_begin;  // per local subdomain
  const int32_t* sub_ntiles;
  int64_t ntiles;                 // all tiles of the rank (partials stride)
  int32_t rev;                    // walk the tiles backwards (alternates between launches so
                                  // each kernel starts on the rows the previous one left in L2)
};

// SELL-32 matrix.  Plain: FP64 values + int32 columns.  Compressed (Z, see
// zformat.cpp): uint8 value codes into `table` + per-(slice, k) int32 column
// base + uint16 offsets.  Both decode to the same entries.
struct Sell {
  const int64_t* sptr;
  const int32_t* col;
  const double* val;
  const int32_t* kbase;  // Z: per slice column k (< 0: -(wide group) - 1)
  const uint16_t* d16;   // Z: column = kbase + d16
  const int32_t* wide;   // Z: int32 columns of wide groups
  const uint8_t* code;   // Z: value = table[code]
  const double* table;
};

// Diagonal of A_p: FP64, or (Z) uint8 codes into the shared value table.
struct Diag {
  const double* v;
  const uint8_t* code;
  const double* table;
};

template <bool Z>
__device__ __forceinline__ double diag_at(const Diag& D, int64_t row) {
  if (Z) return __ldg(&D.table[__ldcs(&D.code[row])]);
  return __ldcs(&D.v[row]);
}

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
  double* partials;      // ntiles * kWarps * kNP
};

// Stop control: sync = one global word (per_sub = 0); async = one word per
// local subdomain (per_sub = 1).
struct Ctl {
  const volatile int32_t* stop;
  int32_t per_sub;
};

// Programmatic dependent launch: let the next kernel of the stream be scheduled
// now, then wait for the full completion (and memory) of the previous kernel.
// Both are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_start() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ bool stopped(const Ctl& C, int lp) {
  return C.stop && C.stop[C.per_sub ? lp : 0];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// The CTA's NV partial sums of tile t (shuffle trees, one CTA barrier, fixed
// order), stored slot-major: partials[j * ntiles + t].  No fence, no atomic:
// the per-subdomain k_finish kernel that follows in stream order reads them.
template <int NV, int NT>
__device__ __forceinline__ void warp_partials(const double (&v)[NV], int64_t t, int64_t ntiles, double* partials) {
  constexpr int NW = NT / 32;
  __shared__ double sh[NV][NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if (lane == 0) sh[j][w] = s;
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double s = warp_sum(lane < NW ? sh[j][lane] : 0.0);
      if (lane == 0) partials[j * ntiles + t] = s;
    }
  }
}

// Sum_k val[e_k] * x[col[e_k]] over SELL-32 row `row` (entries in ascending
// column order as stored).  Matrix data is streamed with evict-first loads so
// the gathered vector keeps its L2 lines.
// W > 0: every slice of the matrix is at most W wide (host-dispatched, fully
// unrolled, predicated on the slice's own width); W == 0: generic loop.
// SMX: x is a shared-memory copy of the columns [xoff, xoff + span).
template <int W, bool Z = false, bool SMX = false>
__device__ __forceinline__ double sell_dot(const Sell& M, int64_t row, const double* x, int32_t xoff = 0) {
  const int64_t s = row >> 5;
  const int lane = (int)(row & 31);
  double acc = 0.0;
  if (Z) {
    // lane-packed SELL-Z (zformat.cpp): W in {4, 8} is the matrix's packed width;
    // one vector load of the row's W codes, one of its W column offsets, and
    // the slice's W column bases (warp-uniform, L1 broadcast).
    static_assert(!Z || W == 4 || W == 8, "SELL-Z widths are 4 or 8");
    uint32_t cw[W / 4 > 0 ? W / 4 : 1];
    uint32_t dw[W / 2 > 0 ? W / 2 : 1];
    int32_t kb[W > 0 ? W : 1];
    if (W == 4) {
      cw[0] = __ldcs(reinterpret_cast<const unsigned int*>(M.code) + row);
      const uint2 d = __ldcs(reinterpret_cast<const uint2*>(M.d16) + row);
      dw[0] = d.x;
      dw[1] = d.y;
      const int4 b = __ldg(reinterpret_cast<const int4*>(M.kbase) + s);
      kb[0] = b.x, kb[1] = b.y, kb[2] = b.z, kb[3] = b.w;
    } else {
      const uint2 c = __ldcs(reinterpret_cast<const uint2*>(M.code) + row);
      cw[0] = c.x;
      cw[W / 4 - 1] = c.y;
      const uint4 d = __ldcs(reinterpret_cast<const uint4*>(M.d16) + row);
      dw[0] = d.x, dw[1] = d.y, dw[2] = d.z, dw[W / 2 - 1] = d.w;
      const int4 b0 = __ldg(reinterpret_cast<const int4*>(M.kbase) + 2 * s);
      const int4 b1 = __ldg(reinterpret_cast<const int4*>(M.kbase) + 2 * s + 1);
      kb[0] = b0.x, kb[1] = b0.y, kb[2] = b0.z, kb[3] = b0.w;
      kb[W - 4] = b1.x, kb[W - 3] = b1.y, kb[W - 2] = b1.z, kb[W - 1] = b1.w;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t code = (cw[k / 4] >> (8 * (k % 4))) & 0xffu;
      const uint32_t off = (dw[k / 2] >> (16 * (k % 2))) & 0xffffu;
      const int32_t c = kb[k] >= 0 ? kb[k] + (int32_t)off : __ldg(&M.wide[(-kb[k] - 1) * 32 + lane]);
      acc += __ldg(&M.table[code]) * (SMX ? x[c - xoff] : __ldg(&x[c]));
    }
    return acc;
  }
  const int64_t base = __ldg(&M.sptr[s]);
  const int w = (int)((__ldg(&M.sptr[s + 1]) - base) >> 5);
  const double* vp = M.val + base + lane;
  const int32_t* cp = M.col + base + lane;
  if (W > 0) {
    double v[W > 0 ? W : 1];
    int32_t c[W > 0 ? W : 1];
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) {
        v[k] = __ldcs(vp + 32 * k);
        c[k] = __ldcs(cp + 32 * k);
      }
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < w) acc += v[k] * (SMX ? x[c[k] - xoff] : __ldg(&x[c[k]]));
  } else {
    for (int k = 0; k < w; ++k) {
      const int32_t c = __ldcs(cp + 32 * k);
      acc += __ldcs(vp + 32 * k) * (SMX ? x[c - xoff] : __ldg(&x[c]));
    }
  }
  return acc;
}

// each kernel defines NT (threads) and RPT = kTileRows / NT (rows per thread)
#define RAS_ROWS_LOOP(j) \
  _Pragma("unroll") for (int j = 0; j < RPT; ++j) if (j * NT + (int)threadIdx.x < ti.y)
#define RAS_ROW(j) ((int64_t)ti.x + j * NT + threadIdx.x)

// ---------------------------------------------------------------------------
// a1+a2: restrict + residual (+ Jacobi PCG start).
//   r = b~ - [A_p|B_p] x (x read in place from owned/halo storage: restrict);
//   JAC: z = D^-1 r, p = z.  Partials: r.z, ||r~||^2, owned ||r~||^2.
// ---------------------------------------------------------------------------
template <bool JAC, int W, bool Z>
static __global__ void __launch_bounds__(Z ? kNT_RES_Z : kNT_RES, Z ? RAS_MB_RES_Z : RAS_MB_RES) k_residual(int64_t tile_base, Tiles T, Sell R,
                                                              const double* __restrict__ b, Diag D,
                                                              const int32_t* __restrict__ own_slot,
                                                              const double* __restrict__ x, double* __restrict__ r,
                                                              double* __restrict__ p, Scal S, Ctl C) {
  constexpr int NT = Z ? kNT_RES_Z : kNT_RES, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  if (stopped(C, ti.z)) return;
  double v[3] = {0.0, 0.0, 0.0};
  double bi[RPT], di[RPT], ax[RPT];
  int32_t os[RPT];
  RAS_ROWS_LOOP(j) {
    bi[j] = __ldcs(&b[RAS_ROW(j)]);
    if (JAC) di[j] = diag_at<Z>(D, RAS_ROW(j));
    os[j] = __ldcs(&own_slot[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) ax[j] = sell_dot<W, Z>(R, RAS_ROW(j), x);
  RAS_ROWS_LOOP(j) {
    const double ri = bi[j] - ax[j];
    r[RAS_ROW(j)] = ri;
    if (JAC) {
      const double zi = __drcp_rn(di[j]) * ri;
      p[RAS_ROW(j)] = zi;
      v[0] += ri * zi;
    }
    v[1] += ri * ri;
    v[2] += os[j] >= 0 ? ri * ri : 0.0;
  }
  warp_partials<3, NT>(v, t, T.ntiles, S.partials);
}

// a3 pass 1: q = A_p p (diag + SELL off-diagonal); partial p.q.
template <int W, bool Z, bool STG>
static __global__ void __launch_bounds__(kNT_SPMV, RAS_MB_SPMV) k_spmv_dot(int64_t tile_base, Tiles T, Sell L, Diag D,
                                                              const double* __restrict__ p, double* __restrict__ q,
                                                              Scal S, Ctl C, const int2* __restrict__ cspan) {
  constexpr int NT = kNT_SPMV, RPT = kTileRows / NT;
  // shared-memory staging of p: a tile whose columns span <= kStageMax rows
  // (2D natural ordering: the tile +- one Omega width) first copies that span of
  // p with coalesced loads, then gathers from shared memory (no dependent L2
  // round trip per neighbour); wider tiles gather from global memory.
  // Measured on B200 (round 1): the barrier after the staging copy serialises
  // the span load and the matrix stream and the halo triples the L2 traffic, so
  // the global-gather path (STG = false) is faster and the default.
  __shared__ double sp[STG ? kStageMax : 1];
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  if (stopped(C, ti.z) || !S.active[ti.z]) return;
  const int2 cs = STG ? cspan[t] : make_int2(0, -1);
  const bool staged = STG && cs.y > 0;
  if (STG) {
    if (staged)
      for (int i = threadIdx.x; i < cs.y; i += NT) sp[i] = __ldg(&p[cs.x + i]);
    __syncthreads();
  }
  double v[1] = {0.0};
  double pi[RPT], di[RPT], ax[RPT];
  RAS_ROWS_LOOP(j) {
    pi[j] = staged ? sp[RAS_ROW(j) - cs.x] : __ldg(&p[RAS_ROW(j)]);
    di[j] = diag_at<Z>(D, RAS_ROW(j));
  }
  if (staged) {
    RAS_ROWS_LOOP(j) ax[j] = sell_dot<W, Z, true>(L, RAS_ROW(j), sp, cs.x);
  } else {
    RAS_ROWS_LOOP(j) ax[j] = sell_dot<W, Z>(L, RAS_ROW(j), p);
  }
  RAS_ROWS_LOOP(j) {
    const double qi = di[j] * pi[j] + ax[j];
    q[RAS_ROW(j)] = qi;
    v[0] += pi[j] * qi;
  }
  warp_partials<1, NT>(v, t, T.ntiles, S.partials);
}

// p_new = z + beta p_old, z = D^-1 r (Jacobi) or z from the trisolves (IC):
// one expression so that a row's own value and its neighbours' recomputation
// of it are bitwise identical.
template <bool IC>
__device__ __forceinline__ double p_next(double g_or_z, double r, double po, double beta, bool first) {
  const double z = IC ? g_or_z : __drcp_rn(g_or_z) * r;
  return first ? z : z + beta * po;
}

// a3 pass 3 of iteration it-1 fused into pass 1 of iteration it (double-
// buffered p): p_new = z + beta p_old for the tile's rows AND, recomputed on
// the fly, for every column it touches; q = A_p p_new; partial p_new.q.
// FIRST (it = 1): p_new = z (beta and p_old unused).
template <int W, bool IC, bool FIRST>
static __global__ void __launch_bounds__(kThreads, 1) k_spmv_pdot(int64_t tile_base, Tiles T, Sell L,
                                                               const double* __restrict__ diag,
                                                               const double* __restrict__ zr,  // r (Jacobi) | z (IC)
                                                               const double* __restrict__ p_old,
                                                               double* __restrict__ p_new, double* __restrict__ q,
                                                               Scal S, Ctl C) {
  constexpr int NT = kThreads, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double beta = FIRST ? 0.0 : S.beta[lp];
  double v[1] = {0.0};
  double pi[RPT], di[RPT], ax[RPT];
  // the gathered arrays stay in L1 (ld.global.nc, L1-allocating): neighbours in
  // the same slice hit the lines this warp just loaded
  for (int j = 0; j < RPT; ++j) {
    const int lr = j * NT + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      di[j] = __ldg(&diag[row]);
      const double a = IC ? __ldg(&zr[row]) : di[j];
      pi[j] = p_next<IC>(a, IC ? 0.0 : __ldg(&zr[row]), FIRST ? 0.0 : __ldg(&p_old[row]), beta, FIRST);
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = j * NT + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      const int64_t s = row >> 5;
      const int lane = (int)(row & 31);
      const int64_t base = __ldg(&L.sptr[s]);
      const int w = (int)((__ldg(&L.sptr[s + 1]) - base) >> 5);
      const double* vp = L.val + base + lane;
      const int32_t* cp = L.col + base + lane;
      double acc = 0.0;
      if (W > 0) {
        double vv[W > 0 ? W : 1];
        int32_t cc[W > 0 ? W : 1];
#pragma unroll
        for (int k = 0; k < W; ++k)
          if (k < w) {
            vv[k] = __ldcs(vp + 32 * k);
            cc[k] = __ldcs(cp + 32 * k);
          }
#pragma unroll
        for (int k = 0; k < W; ++k)
          if (k < w) {
            const int32_t c = cc[k];
            const double gz = IC ? __ldg(&zr[c]) : __ldg(&diag[c]);
            acc += vv[k] * p_next<IC>(gz, IC ? 0.0 : __ldg(&zr[c]), FIRST ? 0.0 : __ldg(&p_old[c]), beta, FIRST);
          }
      } else {
        for (int k = 0; k < w; ++k) {
          const int32_t c = __ldcs(cp + 32 * k);
          const double gz = IC ? __ldg(&zr[c]) : __ldg(&diag[c]);
          acc += __ldcs(vp + 32 * k) *
                 p_next<IC>(gz, IC ? 0.0 : __ldg(&zr[c]), FIRST ? 0.0 : __ldg(&p_old[c]), beta, FIRST);
        }
      }
      ax[j] = acc;
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = j * NT + threadIdx.x;
    if (lr < ti.y) {
      const int64_t row = ti.x + lr;
      const double qi = di[j] * pi[j] + ax[j];
      p_new[row] = pi[j];
      q[row] = qi;
      v[0] += pi[j] * qi;
    }
  }
  warp_partials<1, NT>(v, t, T.ntiles, S.partials);
}

// a3 pass 2: d += alpha p (d = alpha p on the first iteration), r -= alpha q;
// JAC: z = D^-1 r, partials r.z, r.r.  !JAC: partial r.r only.
template <bool JAC, bool Z>
static __global__ void __launch_bounds__(kNT_UPD, RAS_MB_UPD) k_update_dot(int64_t tile_base, Tiles T, Diag D,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ q, double* __restrict__ r,
                                                                double* __restrict__ d, Scal S, Ctl C) {
  constexpr int NT = kNT_UPD, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double alpha = S.alpha[lp];
  const bool first = S.its[lp] == 1;
  double v[2] = {0.0, 0.0};
  double pi[RPT], qi[RPT], ri[RPT], di[RPT], gi[RPT];
  RAS_ROWS_LOOP(j) {
    pi[j] = __ldcs(&p[RAS_ROW(j)]);
    qi[j] = __ldcs(&q[RAS_ROW(j)]);
    ri[j] = __ldcs(&r[RAS_ROW(j)]);
    if (JAC) gi[j] = diag_at<Z>(D, RAS_ROW(j));
    di[j] = first ? 0.0 : __ldcs(&d[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) {
    const double dn = first ? alpha * pi[j] : di[j] + alpha * pi[j];
    const double rn = ri[j] - alpha * qi[j];
    d[RAS_ROW(j)] = dn;
    r[RAS_ROW(j)] = rn;
    if (JAC) v[0] += rn * (__drcp_rn(gi[j]) * rn);
    v[1] += rn * rn;
  }
  warp_partials<2, NT>(v, t, T.ntiles, S.partials);
}

// a3 pass 3 (Jacobi): p = D^-1 r + beta p.
template <bool Z>
static __global__ void __launch_bounds__(kNT_STREAM, RAS_MB_STREAM) k_pupdate(int64_t tile_base, Tiles T, Diag D,
                                                             const double* __restrict__ r, double* __restrict__ p,
                                                             Scal S, Ctl C) {
  constexpr int NT = kNT_STREAM, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double beta = S.beta[lp];
  double gi[RPT], ri[RPT], pi[RPT];
  RAS_ROWS_LOOP(j) {
    gi[j] = diag_at<Z>(D, RAS_ROW(j));
    ri[j] = __ldcs(&r[RAS_ROW(j)]);
    pi[j] = __ldcs(&p[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) p[RAS_ROW(j)] = __drcp_rn(gi[j]) * ri[j] + beta * pi[j];
}

// ---------------------------------------------------------------------------
// Per-subdomain scalar steps of PCG (SURVEY §8c "Exact recurrences"), one CTA
// per subdomain: fixed-order sum of the warp partials of its tiles, then
//   F_RES_JAC : rho = r.z, ||r~||^2, owned ||r~||^2; active = rho != 0 (R7)
//   F_RES_IC  : ||r~||^2, owned ||r~||^2 (rho after z = M^-1 r)
//   F_SPMV    : sigma = p.q; sigma == 0 -> stop (R7) else alpha = rho/sigma, its++
//   F_UPD_JAC : rr; inner stop (||r|| <= eta ||r~||) ; else beta = rho'/rho, rho = rho',
//               stop when its == m or rho' == 0
//   F_UPD_IC  : rr; inner stop; its == m -> stop
//   F_ZDOT0   : rho = r.z, active = rho != 0          (IC path, PCG start)
//   F_ZDOT    : beta = rho'/rho, rho = rho'; rho' == 0 -> stop
// ---------------------------------------------------------------------------
enum FinishOp { F_RES_JAC = 0, F_RES_IC, F_SPMV, F_UPD_JAC, F_UPD_IC, F_ZDOT0, F_ZDOT };

constexpr int kFinThreads = 1024;

template <int OP>
static __global__ void __launch_bounds__(kFinThreads) k_finish(int lp_base, Tiles T, Scal S, Ctl C, int32_t m,
                                                               double inner_tol) {
  constexpr int NV = (OP == F_RES_JAC || OP == F_RES_IC) ? 3 : (OP == F_UPD_JAC || OP == F_UPD_IC) ? 2 : 1;
  constexpr int U = 4;  // independent loads in flight per thread
  __shared__ double sh[NV][kFinThreads / 32];
  const int lp = lp_base + blockIdx.x;
  pdl_start();
  if (stopped(C, lp)) return;
  if (OP != F_RES_JAC && OP != F_RES_IC && !S.active[lp]) return;
  const int64_t base = T.sub_tile_begin[lp];
  const int n = T.sub_ntiles[lp];
  double v[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = 0.0;
  for (int i0 = threadIdx.x; i0 < n; i0 += U * kFinThreads) {
    double a[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * kFinThreads;
#pragma unroll
      for (int j = 0; j < NV; ++j) a[u][j] = i < n ? __ldcg(&S.partials[j * T.ntiles + base + i]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NV; ++j) v[j] += a[u][j];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if (lane == 0) sh[j][w] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double o[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    o[j] = 0.0;
    for (int k = 0; k < kFinThreads / 32; ++k) o[j] += sh[j][k];
  }
  if (OP == F_RES_JAC || OP == F_RES_IC) {
    if (OP == F_RES_JAC) S.rho[lp] = o[0];
    S.rt2[lp] = o[1];
    S.own2[lp] = o[2];
    S.rr[lp] = o[1];
    S.active[lp] = OP == F_RES_JAC ? (o[0] != 0.0) : 1;
    S.its[lp] = 0;
  } else if (OP == F_SPMV) {
    if (o[0] == 0.0) {
      S.active[lp] = 0;
      S.alpha[lp] = 0.0;
    } else {
      S.alpha[lp] = S.rho[lp] / o[0];
      S.its[lp] += 1;
      S.inner_total[lp] += 1;
    }
  } else if (OP == F_UPD_JAC || OP == F_UPD_IC) {
    const double rr = o[NV - 1];
    S.rr[lp] = rr;
    if (inner_tol > 0.0 && sqrt(rr) <= inner_tol * sqrt(S.rt2[lp])) {
      S.active[lp] = 0;  // inner tolerance reached (exact mode / eta)
    } else if (OP == F_UPD_IC) {
      if (S.its[lp] >= m) S.active[lp] = 0;  // z, rho', p of the last iteration are never used
    } else {
      const double rho_new = o[0];
      S.beta[lp] = rho_new / S.rho[lp];
      S.rho[lp] = rho_new;
      if (S.its[lp] >= m || rho_new == 0.0) S.active[lp] = 0;
    }
  } else if (OP == F_ZDOT0) {
    S.rho[lp] = o[0];
    S.active[lp] = o[0] != 0.0;
  } else {  // F_ZDOT
    S.beta[lp] = o[0] / S.rho[lp];
    S.rho[lp] = o[0];
    if (o[0] == 0.0) S.active[lp] = 0;
  }
}

// ---------------------------------------------------------------------------
// a3' (IC(0)/ILU(0)-PCG): M = L U, z = U^-1 L^-1 r by two level-scheduled
// triangular solves (P320-323, level-set strategy).
// ---------------------------------------------------------------------------
#ifndef RAS_TRSV_CHUNK
#define RAS_TRSV_CHUNK 256  // rows per level chunk (factor.cpp) = threads per CTA of k_trsv / _sf / _pf
#endif
constexpr int kTrsvChunk = RAS_TRSV_CHUNK;
#ifndef RAS_TRSV_SLEEP
#define RAS_TRSV_SLEEP 64  // ns between polls of a level counter
#endif

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
static __global__ void __launch_bounds__(kTrsvChunk) k_trsv(TriDev T, int use_batched, int32_t c0, int32_t nchunk,
                                                          uint32_t* counter, int32_t* lev_done,
                                                          const double* __restrict__ in, double* out,
                                                          const int32_t* __restrict__ active, Ctl C) {
  __shared__ int s_c;
  pdl_start();
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
      while (ld_acquire_gpu(done + lev - 1) < need) {
#if RAS_TRSV_SLEEP > 0
        __nanosleep(RAS_TRSV_SLEEP);
#endif
      }
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
      // release: the CTA's out[] stores (ordered before this thread by the barrier)
      // before the count; one fire-and-forget reduction instead of a full
      // sequentially-consistent fence + atomic
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&lev_done[T.sub_lev_off[lp] + lev]) : "memory");
    }
  }
}

// Sync-free variant (round 2): no level barriers.  A CTA claims one chunk (up to
// 256 rows of one level of one subdomain) at a time, in the same topological
// (level) order; each thread solves one row and, for every dependency j, spins
// on out[j] itself until it no longer holds the sentinel --
// the value IS the ready flag (8-byte stores are single-copy atomic), so a
// dependency costs one L2 round trip, not a flag + a value.  The sentinel is a
// signalling-NaN pattern no arithmetic produces (results are quieted).  Sentinel
// hygiene without a reset pass: the forward solve (in r -> out y) re-arms z for
// the backward solve, the backward solve (y -> z) re-arms y for the next forward
// solve, row by row after it read them.  A claimed chunk's dependencies lie in
// earlier claims of running warps, so every spin terminates.
constexpr unsigned long long kTrsvSent = 0xfff4dead0000beefull;
#ifndef RAS_TRSV_SF_SLEEP
#define RAS_TRSV_SF_SLEEP 32  // ns back-off between polls of a dependency
#endif
__device__ __forceinline__ double ld_relaxed_f64_gpu(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64_gpu(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
static __global__ void __launch_bounds__(kTrsvChunk) k_trsv_sf(TriDev T, int use_batched, int32_t c0, int32_t nchunk,
                                                             uint32_t* counter, const double* __restrict__ in,
                                                             double* out, double* rearm,
                                                             const int32_t* __restrict__ active, Ctl C) {
  __shared__ int s_c;
  pdl_start();
  const double sent = __longlong_as_double((long long)kTrsvSent);
  for (;;) {
    // a CTA claims one chunk (<= 256 rows of one level): one row per thread
    if (threadIdx.x == 0) s_c = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int c = s_c;
    __syncthreads();
    if (c >= nchunk) return;
    const int cid = use_batched ? T.batched[c] : c0 + c;
    const int4 ch = T.chunk[cid];
    const bool skip = stopped(C, ch.z) || !active[ch.z];
    const int k = ch.x + threadIdx.x;
    if (k < ch.y) {
      const int32_t i = __ldg(&T.rows[k]);
      const double xin = __ldcg(&in[i]);
      st_relaxed_f64_gpu(&rearm[i], sent);  // the other solve's output, consumed before this launch
      if (!skip) {
        double s = xin;
        const int32_t e1 = __ldg(&T.rp[k + 1]);
        for (int32_t e = __ldg(&T.rp[k]); e < e1; ++e) {
          const double* dep = &out[__ldg(&T.col[e])];
          double v = ld_relaxed_f64_gpu(dep);
          while (__double_as_longlong(v) == (long long)kTrsvSent) {
            __nanosleep(RAS_TRSV_SF_SLEEP);
            v = ld_relaxed_f64_gpu(dep);
          }
          s -= __ldg(&T.val[e]) * v;
        }
        st_relaxed_f64_gpu(&out[i], s / __ldg(&T.diag[i]));
      }
    }
  }
}

// Cluster-resident variant (r2, default when every row has <= 4 dependencies):
// ONE thread-block cluster per subdomain walks that subdomain's levels, the
// level's rows split over the cluster's CTAs (one row per thread, more rows
// only when a level exceeds the cluster's threads).  Between levels the cluster
// meets at the hardware cluster barrier (barrier.cluster arrive.release /
// wait.acquire, ~0.2 us) instead of a level counter in L2 polled by one thread
// per chunk.  The matrix is re-laid out by level-ordered position (row, divisor,
// <= 4 dependency columns padded with -1 and their values: no rp indirection),
// so every static operand of a row is one independent load; rows of levels l+1
// and l+2 are fetched into registers while level l is solved and while the
// cluster barrier is in flight.  The per-level critical path is the barrier
// plus one L2 round trip for the dependencies' values.  Subdomains (clusters)
// never wait on each other.  Same arithmetic and summation order as k_trsv.
constexpr int kNT_TRC = 512;  // 128 registers: two levels x kTrcRPT rows prefetched
struct TriCl {
  const int32_t* lev_pos;      // per subdomain nlev + 1 positions
  const int32_t* sub_pos_off;  // per subdomain offset into lev_pos
  const int32_t* sub_nlev;
  const int32_t* prow;         // per position: row-space row
  const double* pdiv;          // per position: divisor
  const int4* pcol;            // per position: dependency rows, -1 = none
  const double2* pval;         // per position: 2 x (two dependency values)
};
struct TrcRow {
  int32_t i;
  int4 c;
  double in, dv;
  double2 v01, v23;
};
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ int ld_rank0_shared(const int* p) {  // DSMEM read of CTA 0's copy
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  int v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(r) : "memory");
  return v;
}
// static operands of a row (independent loads), then its input value (needs
// the row index: issued one level later, when that index has long arrived)
__device__ __forceinline__ void trc_fetch_static(const TriCl& T, int32_t k, int32_t kend, TrcRow& P) {
  P.i = -1;
  if (k < kend) {
    P.i = __ldg(&T.prow[k]);
    P.dv = __ldg(&T.pdiv[k]);
    P.c = __ldg(&T.pcol[k]);
    P.v01 = __ldg(&T.pval[2 * (int64_t)k]);
    P.v23 = __ldg(&T.pval[2 * (int64_t)k + 1]);
  }
}
__device__ __forceinline__ void trc_fetch_in(const double* __restrict__ in, TrcRow& P) {
  if (P.i >= 0) P.in = __ldg(&in[P.i]);
}
__device__ __forceinline__ void trc_fetch(const TriCl& T, int32_t k, int32_t kend, const double* __restrict__ in,
                                          TrcRow& P) {
  trc_fetch_static(T, k, kend, P);
  trc_fetch_in(in, P);
}
__device__ __forceinline__ void trc_solve(const TrcRow& P, double* out) {
  if (P.i < 0) return;
  // all dependency loads in flight before the first use (L2: written this launch)
  const double o0 = P.c.x >= 0 ? __ldcg(&out[P.c.x]) : 0.0;
  const double o1 = P.c.y >= 0 ? __ldcg(&out[P.c.y]) : 0.0;
  const double o2 = P.c.z >= 0 ? __ldcg(&out[P.c.z]) : 0.0;
  const double o3 = P.c.w >= 0 ? __ldcg(&out[P.c.w]) : 0.0;
  double s = P.in;
  if (P.c.x >= 0) s -= P.v01.x * o0;
  if (P.c.y >= 0) s -= P.v01.y * o1;
  if (P.c.z >= 0) s -= P.v23.x * o2;
  if (P.c.w >= 0) s -= P.v23.y * o3;
  __stcg(&out[P.i], s / P.dv);
}
// one level: the RPT prefetched rows (k0 + u * stride), then (levels wider than
// the cluster's RPT rows per thread) the rest, fetched on the spot
template <int RPT>
__device__ __forceinline__ void trc_level(const TriCl& T, const TrcRow (&P)[RPT], int32_t k0, int32_t kend,
                                          int32_t stride, const double* __restrict__ in, double* out) {
#pragma unroll
  for (int u = 0; u < RPT; ++u) trc_solve(P[u], out);
  for (int32_t k = k0 + RPT * stride; k < kend; k += stride) {
    TrcRow Q;
    trc_fetch(T, k, kend, in, Q);
    trc_solve(Q, out);
  }
}
template <int RPT>
__device__ __forceinline__ void trc_fetch_level(const TriCl& T, int32_t k0, int32_t kend, int32_t stride,
                                                TrcRow (&P)[RPT]) {
#pragma unroll
  for (int u = 0; u < RPT; ++u) trc_fetch_static(T, k0 + u * stride, kend, P[u]);
}
template <int RPT>
__device__ __forceinline__ void trc_fetch_level_in(const double* __restrict__ in, TrcRow (&P)[RPT]) {
#pragma unroll
  for (int u = 0; u < RPT; ++u) trc_fetch_in(in, P[u]);
}
constexpr int kTrcRPT = 2;        // prefetched rows per thread and level
constexpr int kTrcLevSmem = 4096;  // level positions staged in shared memory (more levels: k_trsv)
static __global__ void __launch_bounds__(kNT_TRC, 1) k_trsv_cl(TriCl T, int32_t lp_base, int32_t ntu,
                                                               const double* __restrict__ in, double* out,
                                                               const int32_t* __restrict__ active, Ctl C) {
  constexpr int RPT = kTrcRPT;
  __shared__ int s_skip;
  __shared__ int32_t s_lev[kTrcLevSmem];
  pdl_start();
  const int32_t ncl = (int32_t)cluster_size(), rank = (int32_t)cluster_rank();
  const int lp = lp_base + (int)(blockIdx.x / ncl);
  // the skip decision is CTA 0's, read by all over DSMEM (a stop flag may flip
  // during the launch; the cluster must agree or its barriers would hang)
  if (rank == 0 && threadIdx.x == 0) s_skip = (stopped(C, lp) || !active[lp]) ? 1 : 0;
  const int32_t* glev = T.lev_pos + T.sub_pos_off[lp];
  const int32_t nlev = T.sub_nlev[lp];
  // level positions in shared memory: the cluster barrier's acquire invalidates
  // L1 every level, shared memory stays
  // (the host launches this kernel only when nlev < kTrcLevSmem)
  for (int32_t l = threadIdx.x; l <= nlev; l += kNT_TRC) s_lev[l] = __ldg(&glev[l]);
  cluster_arrive();
  cluster_wait();
  const int skip = ld_rank0_shared(&s_skip);
  cluster_arrive();  // CTA 0 stays until every CTA has read its flag
  cluster_wait();
  if (skip) return;
  const int32_t* lev = s_lev;
  // ntu (<= kNT_TRC) threads per CTA take rows (a test knob; the rest only meet
  // the barriers); thread t of CTA r takes rows lev[l] + (r * ntu + t) + u * stride
  const int32_t stride = ncl * ntu, my = (int32_t)threadIdx.x < ntu ? rank * ntu + (int32_t)threadIdx.x : (1 << 30);
  // software pipeline over levels, in the window between arrive and wait of
  // level l's barrier: the input values of level l+1's rows, the static
  // operands of level l+2's rows
  TrcRow A[RPT], B[RPT];
  trc_fetch_level<RPT>(T, lev[0] + my, lev[1], stride, A);
  trc_fetch_level_in<RPT>(in, A);
#pragma unroll
  for (int u = 0; u < RPT; ++u) B[u].i = -1;
  if (nlev > 1) trc_fetch_level<RPT>(T, lev[1] + my, lev[2], stride, B);
  for (int32_t l = 0; l < nlev; l += 2) {
    trc_level<RPT>(T, A, lev[l] + my, lev[l + 1], stride, in, out);
    cluster_arrive();
    if (l + 1 < nlev) trc_fetch_level_in<RPT>(in, B);
    if (l + 2 < nlev) trc_fetch_level<RPT>(T, lev[l + 2] + my, lev[l + 3], stride, A);
    cluster_wait();
    if (l + 1 < nlev) {
      trc_level<RPT>(T, B, lev[l + 1] + my, lev[l + 2], stride, in, out);
      cluster_arrive();
      if (l + 2 < nlev) trc_fetch_level_in<RPT>(in, A);
      if (l + 3 < nlev) trc_fetch_level<RPT>(T, lev[l + 3] + my, lev[l + 4], stride, B);
      cluster_wait();
    }
  }
}

// Chunk-flag variant with prefetch (r2): k_trsv's chunk schedule (chunks of
// one level claimed in level order; any number of SMs per subdomain) with
// k_trsv_cl's position-ordered operands: after claiming its chunk a thread loads
// its row's static operands and input value BEFORE the wait, so only the
// dependencies' values (L2) remain on the chain.  A chunk waits only for the
// chunks its rows depend on (range [cdep.x, cdep.y] of earlier chunk ids,
// precomputed), not for the whole previous level; flags are cleared before each
// launch and set to `epoch` (1) on completion.  For subdomains whose levels are
// too wide for one cluster (C4: one 256^3 subdomain per GPU).
static __global__ void __launch_bounds__(kTrsvChunk) k_trsv_pf(TriDev T, TriCl P, int use_batched, int32_t c0,
                                                             int32_t nchunk, uint32_t* counter,
                                                             const int2* __restrict__ cdep, int32_t* cflag,
                                                             int32_t epoch, const double* __restrict__ in, double* out,
                                                             const int32_t* __restrict__ active, Ctl C) {
  __shared__ int s_c;
  pdl_start();
  for (;;) {
    if (threadIdx.x == 0) s_c = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int c = s_c;
    __syncthreads();
    if (c >= nchunk) return;
    const int cid = use_batched ? T.batched[c] : c0 + c;
    const int4 ch = T.chunk[cid];
    const int lp = ch.z;
    const bool skip = stopped(C, lp) || !active[lp];
    TrcRow R;
    trc_fetch(P, ch.x + (int32_t)threadIdx.x, skip ? 0 : ch.y, in, R);  // in flight during the wait
    if (!skip && threadIdx.x < 32) {  // one warp polls the producer chunks' flags
      const int2 dr = __ldg(&cdep[cid]);
      for (int32_t d = dr.x + (int32_t)threadIdx.x; d <= dr.y; d += 32)
        while (ld_acquire_gpu(&cflag[d]) != epoch) {
#if RAS_TRSV_SLEEP > 0
          __nanosleep(RAS_TRSV_SLEEP);
#endif
        }
    }
    __syncthreads();
    if (!skip) trc_solve(R, out);
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(&cflag[cid]), "r"(epoch) : "memory");
  }
}

// DSMEM-routed variant (r2, default where it applies): the same cluster-per-
// subdomain level walk, but a row's dependencies never travel through global
// memory.  When row d (level l-1) is solved, its value is pushed straight into
// the shared memory of each CTA that consumes it (another CTA: st.async.
// shared::cluster, completing bytes on that CTA's mbarrier; its own CTA: a plain
// shared store, most consumers of a stencil row); a CTA starts level l once its
// mbarrier has counted all the bytes its level-l rows need from other CTAs.  The cluster still
// meets once per level, but at a RELAXED barrier (no release fence: ~70 ns, and
// no wait for the prefetch loads in flight, which a release's MEMBAR.ALL.GPU
// would wait for -- profiles/r02_trsv_cl_summary.md); it only bounds the skew
// between CTAs to one level, which makes the double-buffered receive slots and
// the mbarrier phases safe.  Applies when every dependency of a level-l row is
// in level l-1 (stencil factors in natural order), a row has <= 4 dependencies
// and <= 4 consumers, and a CTA holds <= kTrdRows rows per thread of a level;
// the routing (consumer CTA, receive slot) is precomputed for a fixed cluster
// size (setup, solver.cu).  Receive slot of dependency q of the row with local
// index j in its CTA's block of the level: j * 4 + q.  Same products in the same
// order as k_trsv: bitwise the same result.
#ifndef RAS_NT_TRD
#define RAS_NT_TRD 512
#endif
constexpr int kNT_TRD = RAS_NT_TRD;  // threads per CTA of k_trsv_ds
constexpr int kTrdRows = 3;                       // rows per thread and level (2 prefetched)
constexpr int kTrdSlots = 4 * kTrdRows * kNT_TRD;  // receive slots per parity
struct TriDs {
  const int32_t* lev_pos;      // per subdomain nlev + 1 positions
  const int32_t* sub_pos_off;  // per subdomain offset into lev_pos
  const int32_t* sub_nlev;
  const int32_t* rb_off;       // per subdomain offset into rbytes
  const int32_t* rbytes;       // per (subdomain, level, CTA): bytes of dependency values the CTA receives
  const int32_t* prow;         // per position: row | ndeps << 29
  const double* pdiv;          // per position: divisor
  const double2* pval;         // per position: 2 x (two dependency values)
  const int4* psend;           // per position: consumers (CTA << 16 | receive slot), -1 = none
};
struct TrdRow {
  uint32_t pr;  // row | ndeps << 29, ~0u = none; decoded only where used (no ALU on a load in flight)
  int4 snd;
  double in, dv;
  double2 v01, v23;
};
constexpr uint32_t kTrdNone = 0xffffffffu;
__device__ __forceinline__ void trd_fetch_static(const TriDs& T, int32_t k, bool ok, TrdRow& P) {
  P.pr = kTrdNone;
  if (ok) {  // predicated loads: the prefetch window issues them and moves on
    P.pr = (uint32_t)__ldg(&T.prow[k]);
    P.dv = __ldg(&T.pdiv[k]);
    P.snd = __ldg(&T.psend[k]);
    P.v01 = __ldg(&T.pval[2 * (int64_t)k]);
    P.v23 = __ldg(&T.pval[2 * (int64_t)k + 1]);
  }
}
__device__ __forceinline__ void trd_fetch_in(const double* __restrict__ in, TrdRow& P) {
  if (P.pr != kTrdNone) P.in = __ldg(&in[P.pr & 0x1fffffffu]);
}
__device__ __forceinline__ void mbar_arm(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_relaxed() {
  __syncthreads();  // the CTA's own plain shared-memory sends, for its consumer threads
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// push v into slot `e & 0xffff` of CTA `e >> 16`'s receive area: another CTA's by
// st.async over DSMEM, completing 8 bytes on its mbarrier mb_next (rcv_next: this
// CTA's address of the area); this CTA's own with a plain shared-memory store
// (ordered for the consumer threads by the CTA barrier that ends the level)
__device__ __forceinline__ void trd_send(int32_t e, double v, double* rcv_local, uint32_t rcv_next, uint32_t mb_next,
                                         uint32_t rank) {
  if (e < 0) return;
  const uint32_t cta = (uint32_t)e >> 16, slot = (uint32_t)e & 0xffffu;
  if (cta == rank) {
    rcv_local[slot] = v;
    return;
  }
  uint32_t ra, rm;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(rcv_next + 8u * slot), "r"(cta));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(mb_next), "r"(cta));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
               "l"(__double_as_longlong(v)), "r"(rm)
               : "memory");
}
__device__ __forceinline__ void trd_solve(const TrdRow& P, const double* rcv_j, double* out, double* rcv_local,
                                          uint32_t rcv_next, uint32_t mb_next, uint32_t rank) {
  if (P.pr == kTrdNone) return;
  const uint32_t nd = P.pr >> 29;
  double s = P.in;
  if (nd > 0) s -= P.v01.x * rcv_j[0];
  if (nd > 1) s -= P.v01.y * rcv_j[1];
  if (nd > 2) s -= P.v23.x * rcv_j[2];
  if (nd > 3) s -= P.v23.y * rcv_j[3];
  const double o = s / P.dv;
  trd_send(P.snd.x, o, rcv_local, rcv_next, mb_next, rank);
  trd_send(P.snd.y, o, rcv_local, rcv_next, mb_next, rank);
  trd_send(P.snd.z, o, rcv_local, rcv_next, mb_next, rank);
  trd_send(P.snd.w, o, rcv_local, rcv_next, mb_next, rank);
  out[P.pr & 0x1fffffffu] = o;  // the result (read by the next kernel)
}
static __global__ void __launch_bounds__(kNT_TRD, 512 / kNT_TRD) k_trsv_ds(TriDs T, int32_t lp_base, const double* __restrict__ in,
                                                               double* out, const int32_t* __restrict__ active, Ctl C) {
  extern __shared__ double rcv[];  // [2][kTrdSlots]
  __shared__ uint64_t mbar[2];
  __shared__ int s_skip;
  __shared__ int2 s_blk[kTrcLevSmem];  // per level: this CTA's block [k0, kend) of positions
  pdl_start();
  const int32_t ncl = (int32_t)cluster_size(), rank = (int32_t)cluster_rank();
  const int lp = lp_base + (int)(blockIdx.x / ncl);
  const int32_t t = (int32_t)threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (rank == 0) s_skip = (stopped(C, lp) || !active[lp]) ? 1 : 0;
  }
  const int32_t* glev = T.lev_pos + T.sub_pos_off[lp];
  const int32_t nlev = T.sub_nlev[lp];
  // level l: CTA r's block = positions b + r q + [0, q), q = ceil(n_l / ncl); row j
  // of the block is thread j % NT's row u = j / NT
  for (int32_t l = t; l < nlev; l += kNT_TRD) {
    const int32_t b = __ldg(&glev[l]), e = __ldg(&glev[l + 1]), q = (e - b + ncl - 1) / ncl;
    s_blk[l] = make_int2(b + rank * q, min(e, b + (rank + 1) * q));
  }
  cluster_arrive();
  cluster_wait();
  const int skip = ld_rank0_shared(&s_skip);
  const int32_t* rb = T.rbytes + T.rb_off[lp];  // [level][ncl]
  if (!skip && t == 0) {  // levels 1 and 2 armed; level l + 2 re-armed after level l
    if (nlev > 1) mbar_arm(&mbar[1], (uint32_t)__ldg(&rb[1 * ncl + rank]));
    if (nlev > 2) mbar_arm(&mbar[0], (uint32_t)__ldg(&rb[2 * ncl + rank]));
  }
  cluster_arrive();  // CTA 0 stays until every CTA has read its flag; every mbarrier initialised
  cluster_wait();
  if (skip) return;
  const uint32_t rcv_s = (uint32_t)__cvta_generic_to_shared(rcv);
  const uint32_t mb_s[2] = {(uint32_t)__cvta_generic_to_shared(&mbar[0]), (uint32_t)__cvta_generic_to_shared(&mbar[1])};
  auto blk = [&](int32_t l, int32_t& k0, int32_t& kend) {
    const int2 bk = s_blk[l];
    k0 = bk.x;
    kend = bk.y;
  };
  auto fetch = [&](int32_t l, TrdRow(&P)[2]) {
    int32_t k0, ke;
    blk(l, k0, ke);
#pragma unroll
    for (int u = 0; u < 2; ++u) trd_fetch_static(T, k0 + u * kNT_TRD + t, k0 + u * kNT_TRD + t < ke, P[u]);
  };
  auto fetch_in = [&](TrdRow(&P)[2]) {
#pragma unroll
    for (int u = 0; u < 2; ++u) trd_fetch_in(in, P[u]);
  };
  auto level = [&](int32_t l, const TrdRow(&P)[2]) {
    const int par = l & 1;
    if (l > 0) mbar_wait(&mbar[par], (uint32_t)(((l - 1) >> 1) & 1));  // phase of level l on mbar[l & 1]
    const double* rc = rcv + par * kTrdSlots;
    double* rl = rcv + (par ^ 1) * kTrdSlots;
    const uint32_t rn = rcv_s + 8u * (uint32_t)((par ^ 1) * kTrdSlots), mn = mb_s[par ^ 1];
#pragma unroll
    for (int u = 0; u < 2; ++u) trd_solve(P[u], rc + 4 * (u * kNT_TRD + t), out, rl, rn, mn, (uint32_t)rank);
    int32_t k0, ke;
    blk(l, k0, ke);
    for (int u = 2; u < kTrdRows; ++u) {  // a third row of a wide level, fetched on the spot
      TrdRow Q;
      trd_fetch_static(T, k0 + u * kNT_TRD + t, k0 + u * kNT_TRD + t < ke, Q);
      trd_fetch_in(in, Q);
      trd_solve(Q, rc + 4 * (u * kNT_TRD + t), out, rl, rn, mn, (uint32_t)rank);
    }
  };
  auto rearm = [&](int32_t l) {  // after the barrier that ended level l - 2 (its phase is over): arm level l
    if (t == 0 && l < nlev) mbar_arm(&mbar[l & 1], (uint32_t)__ldg(&rb[l * ncl + rank]));
  };
  TrdRow A[2], B[2];
  fetch(0, A);
  fetch_in(A);
  B[0].pr = B[1].pr = kTrdNone;
  if (nlev > 1) fetch(1, B);
  for (int32_t l = 0; l < nlev; l += 2) {
    level(l, A);
    if (l + 1 < nlev) fetch_in(B);
    if (l + 2 < nlev) fetch(l + 2, A);
    cluster_sync_relaxed();
    if (l >= 2) rearm(l + 2);  // levels 1 and 2 were armed at the start
    if (l + 1 < nlev) {
      level(l + 1, B);
      if (l + 2 < nlev) fetch_in(A);
      if (l + 3 < nlev) fetch(l + 3, B);
      cluster_sync_relaxed();
      rearm(l + 3);
    }
  }
  cluster_sync_relaxed();  // no CTA leaves while a peer's st.async may still target it
}

// fill with the sync-free trisolve's sentinel (setup, solve start)
static __global__ void k_trsv_arm(int64_t n, double* a, double* b) {
  const double sent = __longlong_as_double((long long)kTrsvSent);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a[i] = sent;
    b[i] = sent;
  }
}

// IC path, after z = M^-1 r: partial r.z (INIT: also p = z).
template <bool INIT>
static __global__ void __launch_bounds__(kNT_STREAM, RAS_MB_STREAM) k_zdot(int64_t tile_base, Tiles T, const double* __restrict__ r,
                                                          const double* __restrict__ z, double* __restrict__ p, Scal S,
                                                          Ctl C) {
  constexpr int NT = kNT_STREAM, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  if (stopped(C, ti.z) || !S.active[ti.z]) return;
  double v[1] = {0.0};
  double ri[RPT], zi[RPT];
  RAS_ROWS_LOOP(j) {
    ri[j] = __ldcs(&r[RAS_ROW(j)]);
    zi[j] = __ldcs(&z[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) {
    v[0] += ri[j] * zi[j];
    if (INIT) p[RAS_ROW(j)] = zi[j];
  }
  warp_partials<1, NT>(v, t, T.ntiles, S.partials);
}

// IC path: p = z + beta p.
static __global__ void __launch_bounds__(kNT_STREAM, RAS_MB_STREAM) k_pupdate_z(int64_t tile_base, Tiles T,
                                                               const double* __restrict__ z, double* __restrict__ p,
                                                               Scal S, Ctl C) {
  constexpr int NT = kNT_STREAM, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  const int lp = ti.z;
  if (stopped(C, lp) || !S.active[lp]) return;
  const double beta = S.beta[lp];
  double zi[RPT], pi[RPT];
  RAS_ROWS_LOOP(j) {
    zi[j] = __ldcs(&z[RAS_ROW(j)]);
    pi[j] = __ldcs(&p[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) p[RAS_ROW(j)] = zi[j] + beta * pi[j];
}

// ---------------------------------------------------------------------------
// Small-subdomain regime (thousands of unknowns per subdomain,
// many subdomains per GPU; the paper's own runs use 4096 per subdomain).  One
// CTA of kNT_SMALL threads runs the WHOLE Jacobi-PCG local solve of one
// subdomain (all m iterations, or to the inner tolerance in exact mode) plus the
// restricted prolongation, with p, r, d in shared memory, q in registers and
// block-level reductions: no per-iteration launches, no host polling.  Same
// recurrences as the tiled path; only summation order differs.
// ---------------------------------------------------------------------------
constexpr int kNT_SMALL = 1024;
constexpr int kSmallMaxRows = 14336;      // p, r in shared memory (16 B / row <= 224 KB)
constexpr int kSmallSmemDRows = 9216;     // up to here d lives in shared memory too (24 B / row), beyond in L2

struct SmallSubs {
  const int32_t* row_off;  // per local subdomain: first row-space row
  const int32_t* nrows;    // padded rows (multiple of 32)
};

// Deterministic block sum of NV values over kNT_SMALL threads; every thread gets the result.
template <int NV>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double (*sh)[kNT_SMALL / 32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if (lane == 0) sh[j][w] = s;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double s = lane < kNT_SMALL / 32 ? sh[j][lane] : 0.0;
    s = warp_sum(s);
    v[j] = __shfl_sync(0xffffffffu, s, 0);
  }
  __syncthreads();
}

// The whole Jacobi-PCG solve of one subdomain by one CTA (kNT_SMALL threads):
// rows [r0, r0 + n) of the row space, p (= z_0), r (= r~) and d in shared
// memory (sp, sr, sd), q in registers; returns the iterations performed.
// Same recurrences as the tiled path; only summation order differs.
template <int RPT, int W, bool Z>
__device__ __forceinline__ int block_pcg(const Sell& L, const Diag& D, int r0, int n, double* sp, double* sr,
                                         double* sd, double rho, double rt2, int m, double inner_tol,
                                         double (*red)[kNT_SMALL / 32]) {
  int its = 0;
  for (;;) {
    // pass 1: q = A_p p, sigma = p.q
    double q[RPT];
    double v1[1] = {0.0};
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int i = j * kNT_SMALL + threadIdx.x;
      if (i < n) {
        const int64_t row = (int64_t)r0 + i;
        q[j] = diag_at<Z>(D, row) * sp[i] + sell_dot<W, Z, true>(L, row, sp, r0);
        v1[0] += sp[i] * q[j];
      }
    }
    block_allsum<1>(v1, red);
    const double sigma = v1[0];
    if (sigma == 0.0) break;  // R7
    const double alpha = rho / sigma;
    ++its;
    // pass 2: d += alpha p, r -= alpha q, z = D^-1 r; r.z, r.r
    double v2[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int i = j * kNT_SMALL + threadIdx.x;
      if (i < n) {
        sd[i] = its == 1 ? alpha * sp[i] : sd[i] + alpha * sp[i];
        const double rn = sr[i] - alpha * q[j];
        sr[i] = rn;
        v2[0] += rn * (__drcp_rn(diag_at<Z>(D, (int64_t)r0 + i)) * rn);
        v2[1] += rn * rn;
      }
    }
    block_allsum<2>(v2, red);
    if (inner_tol > 0.0 && sqrt(v2[1]) <= inner_tol * sqrt(rt2)) break;  // exact mode / eta
    const double beta = v2[0] / rho;
    rho = v2[0];
    if (its >= m || rho == 0.0) break;
    // pass 3: p = z + beta p (own rows only; the previous barrier ended all p reads)
    for (int i = threadIdx.x; i < n; i += kNT_SMALL)
      sp[i] = __drcp_rn(diag_at<Z>(D, (int64_t)r0 + i)) * sr[i] + beta * sp[i];
    __syncthreads();
  }
  return its;
}

// Runs after k_residual<JAC>/k_finish<F_RES_JAC> (r, p = z, rho, rt2, active set).
template <int RPT, int W, bool Z>
static __global__ void __launch_bounds__(kNT_SMALL, 1) k_small_pcg(int lp_base, SmallSubs SS, Sell L, Diag D,
                                                                   const double* __restrict__ r_in,
                                                                   const double* __restrict__ p_in,
                                                                   const int32_t* __restrict__ own_slot,
                                                                   double* __restrict__ x, Scal S, Ctl C, int32_t m,
                                                                   double inner_tol, double* dglob) {
  extern __shared__ double smem[];
  __shared__ double red[2][kNT_SMALL / 32];
  pdl_start();
  const int lp = lp_base + blockIdx.x;
  if (stopped(C, lp) || !S.active[lp]) return;  // uniform per CTA
  const int r0 = SS.row_off[lp], n = SS.nrows[lp];
  double* sp = smem;           // p
  double* sr = smem + n;       // r
  double* sd = dglob ? dglob + r0 : smem + 2 * n;  // d (correction): row-private, shared memory or L2
  for (int i = threadIdx.x; i < n; i += kNT_SMALL) {
    sp[i] = __ldg(&p_in[r0 + i]);
    sr[i] = __ldg(&r_in[r0 + i]);
    sd[i] = 0.0;
  }
  __syncthreads();
  const int its = block_pcg<RPT, W, Z>(L, D, r0, n, sp, sr, sd, S.rho[lp], S.rt2[lp], m, inner_tol, red);
  // a4: restricted prolongation of the owned rows
  if (its > 0)
    for (int i = threadIdx.x; i < n; i += kNT_SMALL) {
      const int32_t s = __ldg(&own_slot[r0 + i]);
      if (s >= 0) x[s] = x[s] + sd[i];
    }
  if (threadIdx.x == 0) {
    S.its[lp] = its;
    S.inner_total[lp] += its;
    S.active[lp] = 0;
  }
}

// ---------------------------------------------------------------------------
// NEXT f1: direct local solve (PAPER §3.3.1, P311-318: factor once, two
// triangular solves per local solve) with the complete banded Cholesky factor
// computed on the host (factor.cpp).  One CTA per subdomain: y = L^-1 r~ then
// d = L^-T y in 32-row blocks, software-pipelined: while warp 0 finishes block
// k (the 32 x 32 coupling to block k-1 and the inverse of the diagonal block,
// both already staged in shared memory: two 32-term dot products per lane,
// no sequential substitution), the other warps compute block k+1's far band sums
// (rows already solved before block k, coalesced along the band rows) and stage
// its coupling / triangle blocks.  One CTA barrier per block.  y / d of the whole
// subdomain live in shared memory; then the restricted prolongation.
// Runs after k_residual / k_finish (r~ in the row space, active set).
// ---------------------------------------------------------------------------
constexpr int kNT_BAND = 512;
constexpr int kBandMaxRows = 12288;  // y / d of one subdomain in shared memory (96 KB)
#ifndef RAS_BAND_PF
#define RAS_BAND_PF 4
#endif
constexpr int kBandPF = RAS_BAND_PF;  // L2 prefetch distance (blocks) of the band rows
constexpr int kStageU = (2048 + (kNT_BAND - 32) - 1) / (kNT_BAND - 32);  // staged block entries per helper thread
constexpr int kStageR = (32 + (kNT_BAND / 32 - 1) - 1) / (kNT_BAND / 32 - 1);  // far-sum rows per helper warp

struct BandDev {
  const double* L;     // lower band, row-major, bw + 1 slots per row (slot j - i + bw)
  const double* U;     // upper band = L^T, row-major (slot j - i)
  const double* binv;  // inverses of the 32 x 32 diagonal blocks of L, [block][32][32] row-major (lower)
  const int64_t* boff; // per local subdomain offset into binv
  const int64_t* off;  // per local subdomain offset into L / U
  const int32_t* bw;   // per local subdomain bandwidth
};

static __global__ void __launch_bounds__(kNT_BAND) k_band_chol(int lp_base, SmallSubs SS, BandDev B,
                                                                 const double* __restrict__ r_in,
                                                                 const int32_t* __restrict__ own_slot,
                                                                 double* __restrict__ x, Scal S, Ctl C) {
  extern __shared__ double sy[];        // y, overwritten by d from the last block down
  __shared__ double blkN[2][32][33];    // coupling of a block's rows to the neighbouring block
  __shared__ double blkT[2][32][33];    // inverse of the block's diagonal triangle (L_kk^-1 or L_kk^-T)
  __shared__ double sv2[32];            // block right-hand side before the triangle (warp 0)
  __shared__ double sfar[2][32];        // rhs minus the far band sums
  pdl_start();
  const int lp = lp_base + blockIdx.x;
  if (stopped(C, lp) || !S.active[lp]) return;
  const int r0 = SS.row_off[lp], n = SS.nrows[lp], nb = n / 32;
  const int b = B.bw[lp];
  const int64_t w = b + 1;
  const double* Lp = B.L + B.off[lp];
  const double* Up = B.U + B.off[lp];
  const double* bip = B.binv + B.boff[lp];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // ---- forward: L y = r~ ----
  // stage block kb (rows i0..i0+31): far sums over columns < i0 - 32, the
  // coupling to block kb-1 and the triangle (helper warps / all warps)
  // t0 / nt: this thread's rank among the staging threads and their count
  // L2 prefetch of the band rows of block kb (one 128-byte line per thread)
  auto prefetch_rows = [&](const double* band, int kb, int t0, int nt) {
    if (kb < 0 || kb >= nb) return;
    const char* base = reinterpret_cast<const char*>(band + (int64_t)kb * 32 * w);
    const int64_t bytes = (int64_t)32 * w * 8;
    for (int64_t o = (int64_t)t0 * 128; o < bytes; o += (int64_t)nt * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
  };
  auto stage_f = [&](int kb, int buf, int t0, int nt) {
    const int i0 = kb * 32;
    prefetch_rows(Lp, kb + kBandPF, t0, nt);  // a later staging reads these from L2
    // coupling to block kb-1 and the triangle: 2 x 32 x 32 independent loads,
    // all issued before any is stored (kStageU per thread)
    double ld[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int t = t0 + u * nt;
      ld[u] = 0.0;
      if (t < 2048) {
        const int l = (t >> 5) & 31, m = t & 31, i = i0 + l;
        if (t < 1024) {
          const int jn = i0 - 32 + m;
          if (kb > 0 && i - jn <= b) ld[u] = __ldg(&Lp[(int64_t)i * w + (jn - i + b)]);
        } else {
          ld[u] = __ldg(&bip[(int64_t)kb * 1024 + l * 32 + m]);  // (L_kk^-1)[l][m]
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int t = t0 + u * nt;
      if (t < 2048) {
        const int l = (t >> 5) & 31, m = t & 31;
        if (t < 1024)
          blkN[buf][l][m] = ld[u];
        else
          blkT[buf][l][m] = ld[u];
      }
    }
    for (int t = t0 + kStageU * nt; t < 2048; t += nt) {  // only when fewer threads stage
      const int l = (t >> 5) & 31, m = t & 31, i = i0 + l;
      if (t < 1024) {
        const int jn = i0 - 32 + m;
        blkN[buf][l][m] = (kb > 0 && i - jn <= b) ? __ldg(&Lp[(int64_t)i * w + (jn - i + b)]) : 0.0;
      } else {
        blkT[buf][l][m] = __ldg(&bip[(int64_t)kb * 1024 + l * 32 + m]);
      }
    }
    // far band sums (columns before block kb-1), one warp per row, the loads of
    // all the warp's rows in flight together
    const int w0 = t0 >> 5, nw = nt >> 5;
    double acc[kStageR];
#pragma unroll
    for (int u = 0; u < kStageR; ++u) {
      acc[u] = 0.0;
      const int l = w0 + u * nw;
      if (l < 32) {
        const int i = i0 + l;
#pragma unroll 4
        for (int j = max(0, i - b) + lane; j < i0 - 32; j += 32) acc[u] += __ldg(&Lp[(int64_t)i * w + (j - i + b)]) * sy[j];
      }
    }
#pragma unroll
    for (int u = 0; u < kStageR; ++u) {
      const int l = w0 + u * nw;
      const double a = warp_sum(acc[u]);
      if (l < 32 && lane == 0) sfar[buf][l] = __ldg(&r_in[r0 + i0 + l]) - a;
    }
    for (int l = w0 + kStageR * nw; l < 32; l += nw) {  // only when fewer warps stage
      const int i = i0 + l;
      double a = 0.0;
      for (int j = max(0, i - b) + lane; j < i0 - 32; j += 32) a += __ldg(&Lp[(int64_t)i * w + (j - i + b)]) * sy[j];
      a = warp_sum(a);
      if (lane == 0) sfar[buf][l] = __ldg(&r_in[r0 + i]) - a;
    }
  };
  for (int k = 1; k < kBandPF; ++k) prefetch_rows(Lp, k, threadIdx.x, kNT_BAND);
  stage_f(0, 0, threadIdx.x, kNT_BAND);
  __syncthreads();
  for (int kb = 0; kb < nb; ++kb) {
    const int cur = kb & 1;
    if (wp == 0) {
      const int i0 = kb * 32;
      // s = rhs - coupling to block kb-1 (four independent partial sums), then
      // y = L_kk^-1 s: a 32-term dot product per lane instead of a 32-step substitution
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      if (kb > 0) {
#pragma unroll
        for (int m = 0; m < 32; ++m) a4[m & 3] += blkN[cur][lane][m] * sy[i0 - 32 + m];
      }
      sv2[lane] = sfar[cur][lane] - ((a4[0] + a4[1]) + (a4[2] + a4[3]));
      __syncwarp();
      double y4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < 32; ++m) y4[m & 3] += blkT[cur][lane][m] * sv2[m];
      sy[i0 + lane] = (y4[0] + y4[1]) + (y4[2] + y4[3]);
      __syncwarp();
    } else if (kb + 1 < nb) {
      stage_f(kb + 1, cur ^ 1, threadIdx.x - 32, kNT_BAND - 32);
    }
    __syncthreads();
  }
  // ---- backward: L^T d = y (block kb's rows of sy hold y until it is solved) ----
  auto stage_b = [&](int kb, int buf, int t0, int nt) {
    const int i0 = kb * 32;
    prefetch_rows(Up, kb - kBandPF, t0, nt);
    double ld[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int t = t0 + u * nt;
      ld[u] = 0.0;
      if (t < 2048) {
        const int l = (t >> 5) & 31, m = t & 31, i = i0 + l;
        if (t < 1024) {
          const int jn = i0 + 32 + m;  // coupling column in block kb+1
          if (kb + 1 < nb && jn - i <= b) ld[u] = __ldg(&Up[(int64_t)i * w + (jn - i)]);
        } else {
          ld[u] = __ldg(&bip[(int64_t)kb * 1024 + m * 32 + l]);  // (L_kk^-T)[l][m] = (L_kk^-1)[m][l]
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int t = t0 + u * nt;
      if (t < 2048) {
        const int l = (t >> 5) & 31, m = t & 31;
        if (t < 1024)
          blkN[buf][l][m] = ld[u];
        else
          blkT[buf][l][m] = ld[u];
      }
    }
    for (int t = t0 + kStageU * nt; t < 2048; t += nt) {
      const int l = (t >> 5) & 31, m = t & 31, i = i0 + l;
      if (t < 1024) {
        const int jn = i0 + 32 + m;
        blkN[buf][l][m] = (kb + 1 < nb && jn - i <= b) ? __ldg(&Up[(int64_t)i * w + (jn - i)]) : 0.0;
      } else {
        blkT[buf][l][m] = __ldg(&bip[(int64_t)kb * 1024 + m * 32 + l]);
      }
    }
    const int w0 = t0 >> 5, nw = nt >> 5;
    double acc[kStageR];
#pragma unroll
    for (int u = 0; u < kStageR; ++u) {
      acc[u] = 0.0;
      const int l = w0 + u * nw;
      if (l < 32) {
        const int i = i0 + l;
        const int j1 = min(n - 1, i + b);
#pragma unroll 4
        for (int j = i0 + 64 + lane; j <= j1; j += 32) acc[u] += __ldg(&Up[(int64_t)i * w + (j - i)]) * sy[j];
      }
    }
#pragma unroll
    for (int u = 0; u < kStageR; ++u) {
      const int l = w0 + u * nw;
      const double a = warp_sum(acc[u]);
      if (l < 32 && lane == 0) sfar[buf][l] = sy[i0 + l] - a;
    }
    for (int l = w0 + kStageR * nw; l < 32; l += nw) {
      const int i = i0 + l;
      double a = 0.0;
      const int j1 = min(n - 1, i + b);
      for (int j = i0 + 64 + lane; j <= j1; j += 32) a += __ldg(&Up[(int64_t)i * w + (j - i)]) * sy[j];
      a = warp_sum(a);
      if (lane == 0) sfar[buf][l] = sy[i] - a;
    }
  };
  for (int k = 1; k < kBandPF; ++k) prefetch_rows(Up, nb - 1 - k, threadIdx.x, kNT_BAND);
  stage_b(nb - 1, (nb - 1) & 1, threadIdx.x, kNT_BAND);
  __syncthreads();
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int cur = kb & 1;
    if (wp == 0) {
      const int i0 = kb * 32;
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      if (kb + 1 < nb) {
#pragma unroll
        for (int m = 0; m < 32; ++m) a4[m & 3] += blkN[cur][lane][m] * sy[i0 + 32 + m];
      }
      sv2[lane] = sfar[cur][lane] - ((a4[0] + a4[1]) + (a4[2] + a4[3]));
      __syncwarp();
      double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < 32; ++m) d4[m & 3] += blkT[cur][lane][m] * sv2[m];
      sy[i0 + lane] = (d4[0] + d4[1]) + (d4[2] + d4[3]);
      __syncwarp();
    } else if (kb > 0) {
      stage_b(kb - 1, cur ^ 1, threadIdx.x - 32, kNT_BAND - 32);
    }
    __syncthreads();
  }
  // a4: restricted prolongation
  for (int i = threadIdx.x; i < n; i += kNT_BAND) {
    const int32_t sl = __ldg(&own_slot[r0 + i]);
    if (sl >= 0) x[sl] = x[sl] + sy[i];
  }
  if (threadIdx.x == 0) {
    S.its[lp] = 1;
    S.active[lp] = 0;
  }
}

// ---------------------------------------------------------------------------
// Grid-resident regime (subdomains of up to ~1.2M rows, e.g. C2's 1024^2 tiles
// + overlap): a persistent cooperative grid, one CTA per SM, split into groups
// of gs CTAs; a group runs the WHOLE Jacobi-PCG local solve of one subdomain
// (then the next one: subdomains lp_base + g, + ngroups, ...) with its rows
// partitioned into contiguous chunks, one per CTA, resident on chip for all m
// iterations: p, r, d and the diagonal codes in shared memory, q in registers.
// HBM is touched once per sweep (r, p in; x[S_p] out; the matrix streams from
// L2), instead of three passes per iteration.
//
// One group-wide reduction per iteration.  PCG's second dot product is taken
// from quantities known before the update (Jacobi, z = D^-1 r):
//   rho' = (r - a q, D^-1 (r - a q)) = rho - 2a (z, q) + a^2 (q, D^-1 q)
//   |r'|^2 = |r|^2 - 2a (r, q) + a^2 (q, q)        (inner tolerance only)
// so sigma = (p, q), (z, q), (q, D^-1 q) [, (r, q), (q, q)] are reduced
// together after the SpMV; the expansion has no cancellation beyond the
// per-iteration ratio rho'/rho (R28).  Same alpha / beta / stop rules
// as the tiled path (R7, R6).
//
// Reductions: no atomics: every CTA stores its partials (after one release
// fence) into its own 32-byte sector of a 3-deep slot ring (the sector of
// reduction k+1 reset to a sentinel before the stores of reduction k), and warp
// 0 of every CTA polls the group's slots with relaxed loads until none holds
// the sentinel, fences once (acquire), then sums them in fixed order -- bitwise-identical
// alpha / beta / stop decisions in all CTAs.  The ring is safe because a CTA
// stores for reduction k only after every CTA finished reading the slots of
// reduction k-2 (it passed reduction k-1).
//
// Halo: the columns of a chunk's rows lie in [-glo, nr + ghi) (host-computed
// ghost zones; only export-band rows reach outside [0, nr): A_p is symmetric).
// At the start of every pass A the ghost rows of p are staged next to the
// chunk's own p in shared memory, so the SpMV gathers from shared memory only.
// A ghost value is recomputed by the reader from values the owner published
// for its export band before the reduction:
//   p_it(c) = fma(beta, p_{it-1}(c), D^-1(c) * fma(-alpha, q_{it-1}(c), r_{it-2}(c)))
// -- the owner's own expression -- so no CTA waits for its neighbours' update.
// Published arrays (export rows only, double-buffered by iteration parity):
// p_it in pub_p[it & 1] (pub_p[1] = k_residual's p = p_1, all rows), r_it in
// pub_r[it & 1] (pub_r[0] = k_residual's r = r_0, all rows), q_it in pub_q[it & 1].
// ---------------------------------------------------------------------------
#ifndef RAS_NT_RESID
#define RAS_NT_RESID 768
#endif
#ifndef RAS_PD_RESID
#define RAS_PD_RESID 1
#endif
constexpr int kNT_RESID = RAS_NT_RESID;
// rows per thread (q in registers, 2 * RPT registers): the largest count the
// register budget of kNT_RESID threads per SM holds without spills
constexpr int kResidMaxRPT = kNT_RESID >= 1024 ? 8 : kNT_RESID >= 832 ? 9 : kNT_RESID >= 768 ? 10 : 16;
constexpr unsigned long long kSlotEmpty = 0xffffffffffffffffull;  // NaN pattern never stored (see group_allsum)
constexpr int kMaxGroupCTAs = 160;  // >= SMs of a B200 (148): CTAs of one group
constexpr int kMaxPat = 128;       // PAT: patterns per chunk table
constexpr int kResidNV = 4;         // slot sector per CTA: up to 4 values per reduction (3 used)

#ifdef RAS_RESID_TRACE
// timing experiment: per CTA, per iteration of the first traced subdomain:
// globaltimer at pass-A start, before the reduction, after it, after pass B
__device__ unsigned long long g_resid_trace[160][64][4];
__device__ unsigned long long g_red_trace[160][64][4];  // per CTA, per reduction: arrive, stored, polled, released
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define RAS_TRACE(slot)                                                                   \
  __syncthreads();                                                                         \
  if (threadIdx.x == 0 && lp == lp_base + 1 && it <= 64) g_resid_trace[blockIdx.x][it - 1][slot] = gtimer();
#else
#define RAS_TRACE(slot)
#endif

struct ResidentCtl {
  const int4* band;           // per (local subdomain, CTA of group), chunk-relative:
                              // {lo_end, hi_begin, glo, ghi}: rows i < lo_end or i >= hi_begin are read
                              // by other CTAs (export band); the chunk's rows reference columns in
                              // [-glo, nr + ghi) (ghost zones, staged in shared memory every iteration)
  unsigned long long* slots;  // per group [3 ring][gs][kResidNV] partial sums, kSlotEmpty before launch
  // row-pattern dictionary (PAT): per chunk (local subdomain, CTA) a table of the
  // distinct rows of A_p -- diagonal + (column delta, value) of each off-diagonal
  // entry, padded to the SELL-Z width W -- and a uint8 pattern id per row
  const int32_t* pat_off;     // per (lp, CTA): first pattern of the chunk's table
  const int32_t* pat_cnt;     // per (lp, CTA): patterns in the table (<= kMaxPat)
  const double* pat_val;      // [pattern][W] off-diagonal values (0 = padding)
  const int32_t* pat_dlt;     // [pattern][W] column - row (0 = padding)
  const double* pat_diag;     // [pattern] diagonal
  const uint8_t* pid;         // row space: pattern id of every row
  double* pub_p[2];           // [1] = k_residual's p (p_1)
  double* pub_r[2];           // [0] = k_residual's r (r_0)
  double* pub_q[2];
  int32_t ngroups, gs;
};

__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// all 32 lanes end with the same bitwise value (xor butterfly: each stage adds
// the same two operands on both partner lanes)
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Group-wide sum of NV values; every thread of every CTA of the group returns
// the identical result.  The CTA's earlier global stores (export band) are
// published by the release store (ordered after them by the CTA barrier);
// readers poll with acquire loads, and the CTA barrier after the poll orders
// every thread's later halo loads after them.  seq = reductions completed.
#ifdef RAS_RESID_TRACE
#define RAS_RTR(k) \
  if (threadIdx.x == 0 && seq < 64) g_red_trace[blockIdx.x][seq][k] = gtimer();
#else
#define RAS_RTR(k)
#endif
template <int NV>
__device__ __forceinline__ void group_allsum(double (&v)[NV], double (*red)[kNT_RESID / 32], double* bc,
                                             unsigned long long* slots, int gs, int c, unsigned& seq) {
  static_assert(NV <= kResidNV, "slot ring holds kResidNV values per CTA");
  constexpr int NW = kNT_RESID / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if (lane == 0) red[j][w] = s;
  }
  __syncthreads();
  RAS_RTR(0)
  if (w == 0) {
    // slots: [3 ring][gs CTAs][4] -- a CTA's values share one 32-byte sector
    unsigned long long* const ring = slots + (size_t)(seq % 3) * gs * 4;
    unsigned long long* const nxt = slots + (size_t)((seq + 1) % 3) * gs * 4;
    double s[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) s[j] = warp_sum(lane < NW ? red[j][lane] : 0.0);
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NV; ++j) st_relaxed_gpu_u64(&nxt[c * 4 + j], kSlotEmpty);
      // release: one fence orders the CTA's earlier stores (export band, ordered
      // before this thread by the CTA barrier) before the value stores
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        unsigned long long u = (unsigned long long)__double_as_longlong(s[j]);
        if (u == kSlotEmpty) u = 0x7ff8000000000000ull;  // a NaN partial stays a NaN, never the sentinel
        st_relaxed_gpu_u64(&ring[c * 4 + j], u);
      }
    }
    RAS_RTR(1)
    // poll: each lane owns CTAs lane, lane + 32, ... and re-loads only the values
    // still empty, all in flight together (relaxed loads; one acquire fence after)
    constexpr int KS = (kMaxGroupCTAs + 31) / 32;
    unsigned long long u[KS][NV];
#pragma unroll
    for (int t = 0; t < KS; ++t)
#pragma unroll
      for (int j = 0; j < NV; ++j) u[t][j] = lane + 32 * t < gs ? kSlotEmpty : 0ull;
    for (;;) {
      bool done = true;
#pragma unroll
      for (int t = 0; t < KS; ++t)
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (u[t][j] == kSlotEmpty) u[t][j] = ld_relaxed_gpu_u64(&ring[(lane + 32 * t) * 4 + j]);
#pragma unroll
      for (int t = 0; t < KS; ++t)
#pragma unroll
        for (int j = 0; j < NV; ++j) done = done && u[t][j] != kSlotEmpty;
      if (__all_sync(0xffffffffu, done)) break;
    }
    RAS_RTR(2)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: the peers' export-band stores
    double acc[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc[j] = 0.0;
#pragma unroll
      for (int t = 0; t < KS; ++t) acc[j] += __longlong_as_double((long long)u[t][j]);  // CTA lane + 32t order
      acc[j] = warp_allsum(acc[j]);
      if (lane == 0) bc[j] = acc[j];
    }
  }
  __syncthreads();
  RAS_RTR(3)
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = bc[j];
  ++seq;
}

// Off-diagonal part of row `row` of the local matrix: sum_k a_k * P(col_k) (SELL-Z
// lane-packed width W in {4, 8}, or plain SELL with W > 0 unrolled / W == 0 loop).
// Z values come from the shared-memory copy of the dictionary `tab`.
template <int W, bool Z, class G>
__device__ __forceinline__ double resident_row(const Sell& L, int64_t row, const double* tab, G P) {
  double acc = 0.0;
  const int64_t sl = row >> 5;
  if (Z) {
    uint32_t cw[W / 4 > 0 ? W / 4 : 1];
    uint32_t dw[W / 2 > 0 ? W / 2 : 1];
    int32_t kb[W > 0 ? W : 1];
    if (W == 4) {
      cw[0] = __ldg(reinterpret_cast<const unsigned int*>(L.code) + row);
      const uint2 dd = __ldg(reinterpret_cast<const uint2*>(L.d16) + row);
      dw[0] = dd.x;
      dw[1] = dd.y;
      const int4 b4 = __ldg(reinterpret_cast<const int4*>(L.kbase) + sl);
      kb[0] = b4.x, kb[1] = b4.y, kb[2] = b4.z, kb[3] = b4.w;
    } else {
      const uint2 cc = __ldg(reinterpret_cast<const uint2*>(L.code) + row);
      cw[0] = cc.x;
      cw[W / 4 - 1] = cc.y;
      const uint4 dd = __ldg(reinterpret_cast<const uint4*>(L.d16) + row);
      dw[0] = dd.x, dw[1] = dd.y, dw[2] = dd.z, dw[W / 2 - 1] = dd.w;
      const int4 b0 = __ldg(reinterpret_cast<const int4*>(L.kbase) + 2 * sl);
      const int4 b1 = __ldg(reinterpret_cast<const int4*>(L.kbase) + 2 * sl + 1);
      kb[0] = b0.x, kb[1] = b0.y, kb[2] = b0.z, kb[3] = b0.w;
      kb[W - 4] = b1.x, kb[W - 3] = b1.y, kb[W - 2] = b1.z, kb[W - 1] = b1.w;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const uint32_t code = (cw[k / 4] >> (8 * (k % 4))) & 0xffu;
      const uint32_t off = (dw[k / 2] >> (16 * (k % 2))) & 0xffffu;
      const int32_t col = kb[k] >= 0 ? kb[k] + (int32_t)off : __ldg(&L.wide[(-kb[k] - 1) * 32 + (row & 31)]);
      acc += tab[code] * P(col);
    }
  } else {
    const int64_t base = __ldg(&L.sptr[sl]);
    const int w = (int)((__ldg(&L.sptr[sl + 1]) - base) >> 5);
    const double* vp = L.val + base + (row & 31);
    const int32_t* cp = L.col + base + (row & 31);
    if (W > 0) {
      double vv[W > 0 ? W : 1];
      int32_t cc[W > 0 ? W : 1];
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k < w) {
          vv[k] = __ldg(vp + 32 * k);
          cc[k] = __ldg(cp + 32 * k);
        }
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k < w) acc += vv[k] * P(cc[k]);
    } else {
      for (int k = 0; k < w; ++k) acc += __ldg(vp + 32 * k) * P(__ldg(cp + 32 * k));
    }
  }
  return acc;
}

// Row-slot order of pass A: 0, RPT-1, 1, RPT-2, ... -- the export bands sit at
// both ends of a chunk, so their published q stores are issued first and have
// completed by the time the reduction's release fence waits for them.
template <int RPT>
__device__ __forceinline__ constexpr int band_first(int jo) {
  return (jo & 1) ? RPT - 1 - (jo >> 1) : (jo >> 1);
}

// Runs after k_residual<JAC>/k_finish<F_RES_JAC> (r, p = z, rho, rt2, active set).
// Launched cooperatively with grid = ngroups * gs CTAs (all co-resident).
// Dynamic shared memory per chunk row: p, r, d (FP64) + the diagonal (Z: uint8
// code into the dictionary and its reciprocals, both copied to shared memory;
// plain: FP64); q lives in registers.  Rows of the export band are the only
// ones with off-chunk columns (A_p is symmetric), so every other row gathers p
// from shared memory without range checks.
template <int RPT, int W, bool Z, bool TOL, bool PAT>
static __global__ void __launch_bounds__(kNT_RESID, 1) k_resident_pcg(int lp_base, int nsub, SmallSubs SS,
                                                                      ResidentCtl RC, Sell L, Diag D,
                                                                      const int32_t* __restrict__ own_slot,
                                                                      double* __restrict__ x, Scal S, Ctl C,
                                                                      int32_t m, double inner_tol, int32_t chunk_max,
                                                                      int32_t glo_max, int32_t ghi_max, int32_t ntable) {
  constexpr int NT = kNT_RESID;
  extern __shared__ double smem[];
  __shared__ double red[kResidNV][NT / 32];
  __shared__ double bc[kResidNV];
  double* sp = smem + glo_max;                  // p of the chunk, ghost zones at [-glo, 0) and [nr, nr + ghi)
  double* sr = smem + glo_max + chunk_max + ghi_max;  // r
  double* sd = sr + chunk_max;        // d (the correction)
  double* stab = sd + chunk_max;      // Z: dictionary values [256]
  double* sinv = stab + 256;          // Z: __drcp_rn of every dictionary value [256]
  uint8_t* sdc = reinterpret_cast<uint8_t*>(sinv + 256);  // Z: diagonal codes (PAT: pattern ids) of the chunk
  double* sdg = stab;                 // plain: diagonal of the chunk
  // PAT: the chunk's pattern table after the ids (8-byte aligned)
  constexpr int WP = W > 0 ? W : 1;
  double* spv = reinterpret_cast<double*>(sdc + ((chunk_max + 7) & ~7));  // [kMaxPat][W] values
  double* spdg = spv + kMaxPat * WP;                                       // [kMaxPat] diagonal
  double* spdi = spdg + kMaxPat;                                           // [kMaxPat] __drcp_rn(diagonal)
  int32_t* spdl = reinterpret_cast<int32_t*>(spdi + kMaxPat);              // [kMaxPat][W] deltas
  static_assert(!PAT || Z, "the row-pattern path needs SELL-Z (ghost pivots come from its dictionary)");
  const int gs = RC.gs;
  const int g = blockIdx.x / gs, c = blockIdx.x - g * gs;
  unsigned long long* slots = RC.slots + (size_t)3 * kResidNV * gs * g;
  unsigned seq = 0;
  // !TOL (fixed m): one reduction of sigma, (z, q), (q, D^-1 q) per iteration.
  // TOL (exact mode / eta): the standard two reductions, sigma then the direct
  // rho' = (r', z'), |r'|^2 -- the expansion above is not used to iterate down
  // to 1e-14 (its rounding drift is not self-correcting).
  constexpr int NV = TOL ? 1 : 3;
  if (Z)
    for (int i = threadIdx.x; i < ntable; i += NT) {
      const double v = __ldg(&D.table[i]);
      stab[i] = v;
      sinv[i] = __drcp_rn(v);
    }
  for (int lp = lp_base + g; lp < lp_base + nsub; lp += RC.ngroups) {
    if (stopped(C, lp) || !S.active[lp]) continue;  // uniform over the group
    const int r0 = SS.row_off[lp], n = SS.nrows[lp];
    const int chunk = ((n / 32 + gs - 1) / gs) * 32;
    const int a = min(n, c * chunk), nr = min(n, a + chunk) - a;
    const int4 band = RC.band[lp * gs + c];
    // chunk row i is row-space row rb + i (rb is a multiple of 32: slice aligned);
    // every array below is re-based to the chunk so indices stay 32-bit
    const int32_t rb = r0 + a;
    // published arrays re-based to the chunk (recomputed where used: registers are scarce)
#define RAS_PUB(arr, par) (((par) ? RC.arr[1] : RC.arr[0]) + rb)  // select, not index: no local-memory copy
    const uint8_t* const dcode = D.code + rb;
    const double* const dval = D.v + rb;
    __syncthreads();
    const int ng = band.z + band.w;  // ghost rows: [-glo, 0) and [nr, nr + ghi)
    auto ghost_row = [&](int t) { return t < band.z ? t - band.z : nr + (t - band.z); };
    for (int t = threadIdx.x; t < ng; t += NT) sp[ghost_row(t)] = __ldcg(&RAS_PUB(pub_p, 1)[ghost_row(t)]);  // p_1
    for (int i = threadIdx.x; i < nr; i += NT) {
      sp[i] = __ldcg(&RAS_PUB(pub_p, 1)[i]);  // p_1 = z_0
      sr[i] = __ldcg(&RAS_PUB(pub_r, 0)[i]);  // r_0
      if (PAT)
        sdc[i] = __ldg(&RC.pid[rb + i]);
      else if (Z)
        sdc[i] = __ldg(&dcode[i]);
      else
        sdg[i] = __ldg(&dval[i]);
    }
    if (PAT) {
      const int p0 = RC.pat_off[lp * gs + c], np = RC.pat_cnt[lp * gs + c];
      for (int t = threadIdx.x; t < np * WP; t += NT) {
        spv[t] = __ldg(&RC.pat_val[(size_t)p0 * WP + t]);
        spdl[t] = __ldg(&RC.pat_dlt[(size_t)p0 * WP + t]);
      }
      for (int t = threadIdx.x; t < np; t += NT) {
        const double dg = __ldg(&RC.pat_diag[p0 + t]);
        spdg[t] = dg;
        spdi[t] = __drcp_rn(dg);  // bitwise the dictionary's reciprocal the ghost readers use
      }
    }
    double q[RPT];
    double rho = S.rho[lp];
    const double rt2 = S.rt2[lp];
    double alpha = 0.0, beta = 0.0;
    int its = 0;
    __syncthreads();
    auto diag = [&](int i) -> double { return PAT ? spdg[sdc[i]] : Z ? stab[sdc[i]] : sdg[i]; };
    auto dinv = [&](int i) -> double { return PAT ? spdi[sdc[i]] : Z ? sinv[sdc[i]] : __drcp_rn(sdg[i]); };
    // Ghost zones of p_{it+1}, staged during pass B of iteration it: the loads of
    // the first kGR ghost rows per thread are issued before pass B (registers),
    // the values p_{it+1}(c) = fma(beta, p_it(c), D^-1(c) fma(-alpha, q_it(c), r_{it-1}(c)))
    // -- the owner's expression -- are stored after it.
    constexpr int kGR = 3;
    double gq[kGR], gr[kGR], gpv[kGR];
    uint32_t gc[kGR];
    auto ghost_issue = [&](int it) {
#pragma unroll
      for (int u = 0; u < kGR; ++u) {
        const int t = threadIdx.x + u * NT;
        if (t < ng) {
          const int li = ghost_row(t);
          gq[u] = __ldcg(&RAS_PUB(pub_q, it & 1)[li]);
          gr[u] = __ldcg(&RAS_PUB(pub_r, (it - 1) & 1)[li]);
          gpv[u] = __ldcg(&RAS_PUB(pub_p, it & 1)[li]);
          if (Z)
            gc[u] = __ldg(&dcode[li]);
          else
            gpv[u] = gpv[u];
        }
      }
    };
    auto ghost_value = [&](int it, int li, double q_, double r_, double p_, uint32_t code) {
      const double di = Z ? sinv[code] : __drcp_rn(__ldg(&dval[li]));
      return __fma_rn(beta, p_, __dmul_rn(di, __fma_rn(-alpha, q_, r_)));
    };
    auto ghost_finish = [&](int it) {
#pragma unroll
      for (int u = 0; u < kGR; ++u) {
        const int t = threadIdx.x + u * NT;
        if (t < ng) sp[ghost_row(t)] = ghost_value(it, ghost_row(t), gq[u], gr[u], gpv[u], Z ? gc[u] : 0u);
      }
      for (int t = threadIdx.x + kGR * NT; t < ng; t += NT) {
        const int li = ghost_row(t);
        sp[li] = ghost_value(it, li, __ldcg(&RAS_PUB(pub_q, it & 1)[li]), __ldcg(&RAS_PUB(pub_r, (it - 1) & 1)[li]),
                             __ldcg(&RAS_PUB(pub_p, it & 1)[li]), Z ? (uint32_t)__ldg(&dcode[li]) : 0u);
      }
    };
    for (;;) {
      const int it = its + 1;
      RAS_TRACE(0)
      // pass A: q = A_p p_it (halo columns recomputed, see above), then the
      // partials sigma = (p, q), (z, q), (q, D^-1 q) [, (r, q), (q, q)]
      double v[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = 0.0;
      auto accum = [&](int j, int i, double pi, double off) {
        const double qi = __fma_rn(diag(i), pi, off);
        q[j] = qi;
        const double di = dinv(i);
        const double zi = __dmul_rn(di, sr[i]);
        const double dq = __dmul_rn(di, qi);
        v[0] += pi * qi;
        if (!TOL) {
          v[NV - 2] += zi * qi;
          v[NV - 1] += qi * dq;
        }
        if (i < band.x || i >= band.y) __stcg(&RAS_PUB(pub_q, it & 1)[i], qi);
      };
      if (PAT) {
        // row patterns: the row's off-diagonal (delta, value) pairs from the
        // chunk's table in shared memory (mostly one pattern per warp: broadcast)
#pragma unroll
        for (int jo = 0; jo < RPT; ++jo) {
          const int j = band_first<RPT>(jo);
          const int i = j * NT + threadIdx.x;
          if (i < nr) {
            const double pi = sp[i];
            const int pt = sdc[i];
            double off = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) off += spv[pt * WP + k] * sp[i + spdl[pt * WP + k]];
            accum(j, i, pi, off);
          }
        }
      } else if (Z) {
        // SELL-Z rows software-pipelined: the codes / offsets / slice bases of
        // row j + PD are in flight while row j is computed (L2 latency hiding)
        constexpr int PD = RPT < RAS_PD_RESID ? RPT : RAS_PD_RESID;
        constexpr int W4 = W / 4 > 0 ? W / 4 : 1, W2 = W / 2 > 0 ? W / 2 : 1, WW = W > 0 ? W : 1;
        const uint8_t* const codeb = L.code + (size_t)rb * W;
        const uint16_t* const d16b = L.d16 + (size_t)rb * W;
        const int32_t* const kbb = L.kbase + (size_t)(rb >> 5) * W;
        uint32_t bcw[PD][W4], bdw[PD][W2];
        int32_t bkb[PD][WW];
        auto zload = [&](int j, int bi) {
          const int i = j * NT + threadIdx.x;
          if (i < nr) {
            if (W == 4) {
              bcw[bi][0] = __ldg(reinterpret_cast<const unsigned int*>(codeb) + i);
              const uint2 dd = __ldg(reinterpret_cast<const uint2*>(d16b) + i);
              bdw[bi][0] = dd.x;
              bdw[bi][W2 - 1] = dd.y;
              const int4 b4 = __ldg(reinterpret_cast<const int4*>(kbb) + (i >> 5));
              bkb[bi][0] = b4.x, bkb[bi][1] = b4.y, bkb[bi][2] = b4.z, bkb[bi][WW - 1] = b4.w;
            } else {
              const uint2 cc = __ldg(reinterpret_cast<const uint2*>(codeb) + i);
              bcw[bi][0] = cc.x;
              bcw[bi][W4 - 1] = cc.y;
              const uint4 dd = __ldg(reinterpret_cast<const uint4*>(d16b) + i);
              bdw[bi][0] = dd.x, bdw[bi][1] = dd.y, bdw[bi][2] = dd.z, bdw[bi][W2 - 1] = dd.w;
              const int4 b0 = __ldg(reinterpret_cast<const int4*>(kbb) + 2 * (i >> 5));
              const int4 b1 = __ldg(reinterpret_cast<const int4*>(kbb) + 2 * (i >> 5) + 1);
              bkb[bi][0] = b0.x, bkb[bi][1] = b0.y, bkb[bi][2] = b0.z, bkb[bi][3] = b0.w;
              bkb[bi][WW - 4] = b1.x, bkb[bi][WW - 3] = b1.y, bkb[bi][WW - 2] = b1.z, bkb[bi][WW - 1] = b1.w;
            }
          }
        };
#pragma unroll
        for (int j = 0; j < PD; ++j) zload(band_first<RPT>(j), j);
#pragma unroll
        for (int jo = 0; jo < RPT; ++jo) {
          const int j = band_first<RPT>(jo);
          const int i = j * NT + threadIdx.x;
          const int bi = jo % PD;
          if (i < nr) {
            const double pi = sp[i];
            // a slice with a wide group (base < 0: int32 columns) takes the generic decoder
            bool wide = false;
#pragma unroll
            for (int k = 0; k < W; ++k) wide = wide || bkb[bi][k] < 0;
            double off = 0.0;
            if (!wide) {
#pragma unroll
              for (int k = 0; k < W; ++k) {
                const uint32_t code = (bcw[bi][k / 4] >> (8 * (k % 4))) & 0xffu;
                const int li = bkb[bi][k] - rb + (int)((bdw[bi][k / 2] >> (16 * (k % 2))) & 0xffffu);
                off += stab[code] * sp[li];
              }
            } else {
              off = resident_row<W, Z>(L, (int64_t)rb + i, stab, [&](int32_t col) { return sp[col - rb]; });
            }
            accum(j, i, pi, off);
          }
          if (jo + PD < RPT) zload(band_first<RPT>(jo + PD), bi);
        }
      } else {
#pragma unroll
        for (int jo = 0; jo < RPT; ++jo) {
          const int j = band_first<RPT>(jo);
          const int i = j * NT + threadIdx.x;
          if (i < nr) {
            const double pi = sp[i];
            const double off = resident_row<W, Z>(L, (int64_t)rb + i, stab, [&](int32_t col) { return sp[col - rb]; });
            accum(j, i, pi, off);
          }
        }
      }
      RAS_TRACE(1)
      group_allsum<NV>(v, red, bc, slots, gs, c, seq);
      RAS_TRACE(2)
      const double sigma = v[0];
      if (sigma == 0.0) break;  // R7
      alpha = rho / sigma;
      its = it;
      bool stop;
      if (!TOL) {
        const double rho_new = rho - 2.0 * alpha * v[NV - 2] + alpha * alpha * v[NV - 1];
        stop = its >= m || !(rho_new > 0.0);  // R7 (rho' <= 0 only by rounding: breakdown)
        beta = rho_new / rho;
        rho = rho_new;
        if (!stop) ghost_issue(it);
        // pass B (own rows): d += alpha p, r -= alpha q, and unless stopping
        // p_{it+1} = D^-1 r + beta p; publish r_it, p_{it+1} of the export band
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int i = j * NT + threadIdx.x;
          if (i < nr) {
            const double pi = sp[i];
            sd[i] = it == 1 ? alpha * pi : __fma_rn(alpha, pi, sd[i]);
            if (!stop) {
              const double rn = __fma_rn(-alpha, q[j], sr[i]);
              sr[i] = rn;
              const double pn = __fma_rn(beta, pi, __dmul_rn(dinv(i), rn));
              sp[i] = pn;
              if (i < band.x || i >= band.y) {
                __stcg(&RAS_PUB(pub_r, it & 1)[i], rn);
                __stcg(&RAS_PUB(pub_p, (it + 1) & 1)[i], pn);
              }
            }
          }
        }
        if (!stop) ghost_finish(it);
      } else {
        // pass B1: d += alpha p, r -= alpha q (published), z = D^-1 r; (r, z), (r, r)
        double v2[2] = {0.0, 0.0};
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int i = j * NT + threadIdx.x;
          if (i < nr) {
            const double pi = sp[i];
            sd[i] = it == 1 ? alpha * pi : __fma_rn(alpha, pi, sd[i]);
            const double rn = __fma_rn(-alpha, q[j], sr[i]);
            sr[i] = rn;
            const double zi = __dmul_rn(dinv(i), rn);
            v2[0] += rn * zi;
            v2[1] += rn * rn;
            if (i < band.x || i >= band.y) __stcg(&RAS_PUB(pub_r, it & 1)[i], rn);
          }
        }
        group_allsum<2>(v2, red, bc, slots, gs, c, seq);
        stop = its >= m || v2[0] == 0.0 || sqrt(v2[1]) <= inner_tol * sqrt(rt2);  // R7, R6
        beta = v2[0] / rho;
        rho = v2[0];
        if (!stop) ghost_issue(it);
        // pass B2: p_{it+1} = D^-1 r + beta p (published)
        if (!stop) {
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            const int i = j * NT + threadIdx.x;
            if (i < nr) {
              const double pn = __fma_rn(beta, sp[i], __dmul_rn(dinv(i), sr[i]));
              sp[i] = pn;
              if (i < band.x || i >= band.y) __stcg(&RAS_PUB(pub_p, (it + 1) & 1)[i], pn);
            }
          }
          ghost_finish(it);
        }
      }
      RAS_TRACE(3)
      if (stop) break;
      __syncthreads();
    }
    // a4: restricted prolongation of the chunk's owned rows
    __syncthreads();
    if (its > 0) {
      for (int i = threadIdx.x; i < nr; i += NT) {
        const int32_t s = __ldg(&own_slot[rb + i]);
        if (s >= 0) x[s] = x[s] + sd[i];
      }
    }
    if (c == 0 && threadIdx.x == 0) {
      S.its[lp] = its;
      S.inner_total[lp] += its;
      S.active[lp] = 0;
    }
#undef RAS_PUB
  }
}

// a4: restricted prolongation x[S_p] += d[S_p] (overlap part of d discarded).
static __global__ void __launch_bounds__(kNT_STREAM, RAS_MB_STREAM) k_prolong(int64_t tile_base, Tiles T,
                                                             const int32_t* __restrict__ own_slot,
                                                             const double* __restrict__ d, double* __restrict__ x,
                                                             Scal S, Ctl C) {
  constexpr int NT = kNT_STREAM, RPT = kTileRows / NT;
  pdl_start();
  const int64_t t = tile_base + (T.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x);
  const int4 ti = T.tile[t];
  if (stopped(C, ti.z) || S.its[ti.z] == 0) return;  // no PCG step taken: d == 0
  int32_t os[RPT];
  double di[RPT];
  RAS_ROWS_LOOP(j) {
    os[j] = __ldcs(&own_slot[RAS_ROW(j)]);
    di[j] = __ldcs(&d[RAS_ROW(j)]);
  }
  RAS_ROWS_LOOP(j) if (os[j] >= 0) x[os[j]] = x[os[j]] + di[j];
}

#undef RAS_ROWS_LOOP
#undef RAS_ROW

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

// every rank's owned values, allgathered in padded per-rank segments -> global
// order (x_out gather on N GPUs, P242); padding slots carry gid -1
static __global__ void k_gather_all(int64_t count, const int32_t* __restrict__ gid_all, const double* __restrict__ v,
                                    double* __restrict__ xg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = gid_all[i];
    if (g >= 0) xg[g] = v[i];
  }
}

// owned storage -> global order (x_out gather, P242)
static __global__ void k_gather_x(int64_t n_own, const int32_t* __restrict__ own_gid, const double* __restrict__ x,
                                  double* __restrict__ xg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_own; i += (int64_t)gridDim.x * blockDim.x)
    xg[own_gid[i]] = x[i];
}

}  // namespace ras
