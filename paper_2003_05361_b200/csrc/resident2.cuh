// RESIDENT path, version 2 (k_resident2): the on-chip fixed-m Jacobi-PCG of
// k_resident_pcg (same recurrences R28 / R29, same row-pattern dictionary SpMV,
// bitwise the same iterates) with the per-thread vectors r and d moved from
// shared memory into TENSOR MEMORY (TMEM, 256 KB per SM, used here as a private
// register-file extension: tcgen05.st / tcgen05.ld of 32-bit columns of the
// thread's own TMEM lane) and NL subdomains interleaved per CTA.
//
// Why (profiles/r01_resident_ncu_summary.md): k_resident_pcg runs
// one group-wide reduction per PCG iteration whose latency (~3.9 us at 148 CTAs)
// is about a third of the iteration, and its shared memory (p, r, d: 24 B/row +
// ghosts) caps a CTA's chunk at ~7.7 K rows.  With r and d in TMEM a chunk row
// costs 9 B of shared memory (p + pattern id), so
//   NL = 2: two subdomains live on chip at once and the reduction of one is in
//           flight while the CTA runs the other's passes (software pipelining
//           across independent local problems -- the subdomains of a sweep);
//   NL = 1: chunks up to 768 x 16 rows (C5's 1.56 M-row Voronoi cells on 148 SMs).
//
// Per lane (subdomain) L and iteration it, exactly as k_resident_pcg:
//   pass A   q = A_p p_it (pattern SpMV from shared memory), partials
//            (p, q), (z, q), (q, D^-1 q); publish them (slot ring, no wait)
//   wait     the lane's group-wide sum -> alpha, rho' (R28), beta
//   pass B   d += alpha p, r -= alpha q, p_{it+1} = D^-1 r + beta p; export band
//            published; ghost zones recomputed (R29)
// Schedule with NL = 2: A(0) pub(0) A(1) pub(1) | wait(0) B(0) A(0) pub(0) wait(1) B(1) A(1) pub(1) | ...
//
// TMEM layout: warp w addresses the 32 lanes of quadrant w % 4 (its lane = its
// thread's lane), columns [kR2ColBlk * (w / 4), +kR2ColBlk); thread column
// ((L * 2 + V) * RPT + j) * 2 holds vector V (0 = r, 1 = d) of chunk row
// j * NT + tid of lane L as two 32-bit halves.  tcgen05.ld/st are warp-wide
// (.sync.aligned): they are executed unconditionally, also for rows past the
// chunk end (private slots, harmless).
#pragma once

namespace ras {

constexpr int kNT_R2 = 512;     // threads per CTA: 16 warps, 4 per TMEM lane quadrant, 128 registers per thread
constexpr int kR2ColBlk = 128;  // TMEM columns per warp (4 warps per quadrant: 512 columns)
constexpr int kR2MaxRPT = 24;   // rows per thread of one lane (q in registers)

__device__ __forceinline__ void tm_st(uint32_t taddr, double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"((uint32_t)u),
               "r"((uint32_t)(u >> 32))
               : "memory");
}
__device__ __forceinline__ double tm_ld(uint32_t taddr) {
  uint32_t lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}
__device__ __forceinline__ void tm_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// First half of group_allsum: CTA partials -> this CTA's slot of reduction `seq`
// (the next ring sector reset first, one release fence, relaxed stores).
template <int NV, int NT>
__device__ __forceinline__ void group_publish(const double (&v)[NV], double (*red)[NT / 32],
                                              unsigned long long* slots, int gs, int c, unsigned seq) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double s = warp_sum(v[j]);
    if (lane == 0) red[j][w] = s;
  }
  __syncthreads();
  if (w == 0) {
    unsigned long long* const ring = slots + (size_t)(seq % 3) * gs * 4;
    unsigned long long* const nxt = slots + (size_t)((seq + 1) % 3) * gs * 4;
    double s[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) s[j] = warp_sum(lane < NW ? red[j][lane] : 0.0);
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NV; ++j) st_relaxed_gpu_u64(&nxt[c * 4 + j], kSlotEmpty);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release: export-band stores before the values
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        unsigned long long u = (unsigned long long)__double_as_longlong(s[j]);
        if (u == kSlotEmpty) u = 0x7ff8000000000000ull;
        st_relaxed_gpu_u64(&ring[c * 4 + j], u);
      }
    }
  }
  // red[] is reused by the next publish only after a later CTA barrier
}

// Second half: poll every CTA's slot of reduction `seq`, fixed-order sum; every
// thread returns the identical values.
template <int NV>
__device__ __forceinline__ void group_wait(double (&v)[NV], double* bc, const unsigned long long* slots, int gs,
                                           unsigned seq) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {
    const unsigned long long* const ring = slots + (size_t)(seq % 3) * gs * 4;
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
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: the peers' export-band stores
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < KS; ++t) acc += __longlong_as_double((long long)u[t][j]);
      acc = warp_allsum(acc);
      if (lane == 0) bc[j] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = bc[j];
}

// Shared-memory words (doubles) of one lane: p with ghost zones, pattern ids,
// pattern table (values [kMaxPat][W], diagonal, its reciprocal, int32 deltas [kMaxPat][W]).
// PAT: + the pattern table; !PAT: + the chunk's SELL-Z slice bases (int32 [slices][W]).
__host__ __device__ constexpr int r2_lane_words(int glo, int chunk, int ghi, int W, bool pat) {
  return (glo + chunk + ghi) + ((chunk + 7) & ~7) / 8 +
         (pat ? kMaxPat * (W + 2) + (kMaxPat * W + 1) / 2 : ((chunk + 31) / 32 * W + 1) / 2);
}

// Off-diagonal sum of a SELL-Z row whose slice has a wide group (int32 columns):
// the generic decoder, out of line so its registers do not burden the hot loop.
template <int W>
__device__ __noinline__ double r2_wide_row(const Sell& L, int64_t row, const double* tab, const double* p_rowspace) {
  return resident_row<W, true>(L, row, tab, [&](int32_t col) { return p_rowspace[col]; });
}

// Per-lane state kept in shared memory (registers are for the rows' q).
struct R2Lane {
  int lp, rb, nr, live;  // subdomain, chunk's first row-space row, chunk rows, still iterating
  int4 band;             // {lo_end, hi_begin, glo, ghi}
  double rho, alpha, beta;
  int its;
  unsigned seq;
};

// Named barriers (id 0 is __syncthreads): compute warps only; partials of lane
// L ready (compute arrive, reduction warp waits); result of lane L ready
// (reduction warp arrives, compute warps wait).
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
constexpr int kBarCompute = 1;
__device__ __forceinline__ int bar_part(int L) { return 2 + L; }
__device__ __forceinline__ int bar_res(int L) { return 4 + L; }

// four consecutive TMEM doubles (8 columns) of this thread's lane
__device__ __forceinline__ void tm_ld4(uint32_t taddr, double (&v)[4]) {
  uint32_t a[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = __longlong_as_double((long long)(((unsigned long long)a[2 * k + 1] << 32) | a[2 * k]));
}
__device__ __forceinline__ void tm_st4(uint32_t taddr, const double (&v)[4]) {
  uint32_t a[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v[k]);
    a[2 * k] = (uint32_t)u;
    a[2 * k + 1] = (uint32_t)(u >> 32);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a[0]),
               "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Warp-specialised CTA: warp 0 is the REDUCTION warp (sums the compute warps'
// partials, publishes them to the group's slot ring, polls it, computes alpha /
// beta / the stop decision); warps 1..15 are COMPUTE warps (rows j * kNC + ct,
// ct = threadIdx.x - 32).  They meet only at named barriers, so the compute warps
// never wait for the release fence or the poll of a reduction they do not need yet.
constexpr int kNC_R2 = kNT_R2 - 32;  // compute threads

// PAT: row-pattern dictionary SpMV (stencil matrices: <= kMaxPat distinct rows per
// chunk, no matrix stream); !PAT: the SELL-Z local matrix streamed from L2 every
// iteration (codes / column offsets / slice bases; irregular subdomains such as
// Voronoi cells, whose chunks hold hundreds of distinct rows), one batch of four
// rows' entries in flight while the previous batch is computed.
template <int RPT, int W, int NL, bool PAT>
static __global__ void __launch_bounds__(kNT_R2, 1) k_resident2(int lp_base, int nsub, SmallSubs SS, ResidentCtl RC,
                                                                   Sell Lm, Diag D, const int32_t* __restrict__ own_slot,
                                                                   double* __restrict__ x, Scal S, Ctl C, int32_t m,
                                                                   int32_t chunk_max, int32_t glo_max, int32_t ghi_max,
                                                                   int32_t ntable) {
  constexpr int NT = kNT_R2, NC = kNC_R2, NCW = NC / 32;
  static_assert(RPT % 4 == 0, "TMEM rows move in groups of four");
  static_assert(2 * 2 * NL * RPT <= kR2ColBlk, "r, d of NL lanes x RPT rows must fit the warp's TMEM columns");
  extern __shared__ double smem[];
  __shared__ double red[NL][3][NCW];  // compute warps' partials per lane
  __shared__ double sinv[256];         // __drcp_rn of every dictionary value (ghost rows' D^-1)
  __shared__ double stab[256];         // !PAT: the dictionary values (matrix entries and diagonal)
  __shared__ R2Lane st[NL];
  __shared__ uint32_t s_tbase;
  // per-lane shared memory: p (+ ghost zones) | pattern ids | pattern table
  const int pstride = glo_max + chunk_max + ghi_max;
  const int idbytes = (chunk_max + 7) & ~7;
  const int lane_words = r2_lane_words(glo_max, chunk_max, ghi_max, W, PAT);
  auto lane_sp = [&](int L) { return smem + (size_t)L * lane_words + glo_max; };
  auto lane_id = [&](int L) { return reinterpret_cast<uint8_t*>(smem + (size_t)L * lane_words + pstride); };
  auto lane_pv = [&](int L) { return smem + (size_t)L * lane_words + pstride + idbytes / 8; };  // [kMaxPat][W]
  auto lane_pdg = [&](int L) { return lane_pv(L) + kMaxPat * W; };
  auto lane_pdi = [&](int L) { return lane_pdg(L) + kMaxPat; };
  auto lane_pdl = [&](int L) { return reinterpret_cast<int32_t*>(lane_pdi(L) + kMaxPat); };  // [kMaxPat][W]
  auto lane_kb = [&](int L) { return reinterpret_cast<int32_t*>(lane_pv(L)); };  // !PAT: [slices][W] slice bases
  const int gmax = glo_max + ghi_max;
  double* const sstage = smem + (size_t)NL * lane_words;  // ghost staging: q [gmax] | r [gmax]

  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ct = threadIdx.x - 32;  // compute thread index (< 0 in the reduction warp)
  // ---- TMEM: 512 columns for this CTA (one CTA per SM) ----
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < ntable; i += NT) {
    const double v = __ldg(&D.table[i]);
    stab[i] = v;
    sinv[i] = __drcp_rn(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmy = s_tbase + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(kR2ColBlk * (w >> 2));
  auto tcol = [&](int L, int V, int j) { return tmy + (uint32_t)(((L * 2 + V) * RPT + j) * 2); };

  const int gs = RC.gs;
  const int g = blockIdx.x / gs, c = blockIdx.x - g * gs;
  auto lane_slots = [&](int L) { return RC.slots + (size_t)3 * kResidNV * gs * (g * NL + L); };

  // published arrays re-based to a chunk (select, not index)
#define R2_PUB(arr, par, rb) (((par) ? RC.arr[1] : RC.arr[0]) + (rb))

  // reduction counters run over the whole launch (like k_resident_pcg's): the
  // 3-deep slot ring of a lane is only safe while every CTA agrees on its position
  if (threadIdx.x < NL) st[threadIdx.x].seq = 0;
  for (int pair = g; pair * NL < nsub; pair += RC.ngroups) {
    // ---- lane set-up (all warps): p_1, r_0, pattern ids and the chunk's pattern table ----
    bool live[NL];
#pragma unroll
    for (int L = 0; L < NL; ++L) {
      const int lp = lp_base + pair * NL + L;
      __syncthreads();
      if (threadIdx.x == 0) {
        const bool valid = pair * NL + L < nsub;
        st[L].lp = lp;
        st[L].live = valid && !stopped(C, lp) && S.active[lp];
        st[L].its = 0;
        st[L].alpha = st[L].beta = 0.0;
        if (st[L].live) {
          const int r0 = SS.row_off[lp], n = SS.nrows[lp];
          const int chunk = ((n / 32 + gs - 1) / gs) * 32;
          const int a = min(n, c * chunk);
          st[L].rb = r0 + a;
          st[L].nr = min(n, a + chunk) - a;
          st[L].band = RC.band[lp * gs + c];
          st[L].rho = S.rho[lp];
        }
      }
      __syncthreads();
      live[L] = st[L].live;
      if (!live[L]) continue;
      const int rb = st[L].rb, nr = st[L].nr;
      const int4 band = st[L].band;
      double* sp = lane_sp(L);
      uint8_t* sdc = lane_id(L);
      const int ng = band.z + band.w;
      for (int t = threadIdx.x; t < ng; t += NT) {
        const int li = t < band.z ? t - band.z : nr + (t - band.z);
        sp[li] = __ldcg(&R2_PUB(pub_p, 1, rb)[li]);  // p_1 of the ghost rows
      }
      for (int i = threadIdx.x; i < nr; i += NT) {
        sp[i] = __ldcg(&R2_PUB(pub_p, 1, rb)[i]);  // p_1 = z_0
        sdc[i] = PAT ? __ldg(&RC.pid[rb + i]) : __ldg(&D.code[rb + i]);  // pattern id | diagonal code
      }
      if (ct >= 0) {
#pragma unroll
        for (int b = 0; b < RPT / 4; ++b) {
          double rr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = (4 * b + u) * NC + ct;
            rr[u] = i < nr ? __ldcg(&R2_PUB(pub_r, 0, rb)[i]) : 0.0;  // r_0
          }
          tm_st4(tcol(L, 0, 4 * b), rr);
        }
      }
      const int p0 = PAT ? RC.pat_off[lp * gs + c] : 0, np = PAT ? RC.pat_cnt[lp * gs + c] : 0;
      double* spv = lane_pv(L);
      int32_t* spdl = lane_pdl(L);
      for (int t = threadIdx.x; t < np * W; t += NT) {
        spv[t] = __ldg(&RC.pat_val[(size_t)p0 * W + t]);
        spdl[t] = __ldg(&RC.pat_dlt[(size_t)p0 * W + t]);
      }
      for (int t = threadIdx.x; t < np; t += NT) {
        const double dg = __ldg(&RC.pat_diag[p0 + t]);
        lane_pdg(L)[t] = dg;
        lane_pdi(L)[t] = __drcp_rn(dg);
      }
      if (!PAT) {
        int32_t* skb = lane_kb(L);
        for (int t = threadIdx.x; t < (nr + 31) / 32 * W; t += NT) skb[t] = __ldg(&Lm.kbase[(size_t)(rb >> 5) * W + t]);
      }
    }
    tm_st_wait();
    __syncthreads();

    if (w == 0) {
      // ================= reduction warp =================
      // The compute warps run, per live lane L in turn: sync RES(L); pass B;
      // pass A; arrive PART(L) -- and then immediately need RES(next lane).  So
      // on PART(L) this warp first releases RES(next) (polled while the compute
      // warps were busy with L), then publishes L's partials, then polls the next
      // result it will need: the compute warps never wait for a fence or a poll.
      double part[3];
      auto take_part = [&](int L) {  // the compute warps' partials of lane L
        nbar_sync(bar_part(L), NT);
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) part[j2] = warp_sum(lane < NCW ? red[L][j2][lane] : 0.0);
      };
      auto publish = [&](int L) {  // part -> this CTA's slot of the lane's current reduction
        unsigned long long* slots = lane_slots(L);
        const unsigned seq = st[L].seq;
        unsigned long long* const ring = slots + (size_t)(seq % 3) * gs * 4;
        unsigned long long* const nxt = slots + (size_t)((seq + 1) % 3) * gs * 4;
        if (lane == 0) {
#pragma unroll
          for (int j2 = 0; j2 < 3; ++j2) st_relaxed_gpu_u64(&nxt[c * 4 + j2], kSlotEmpty);
          // release: the compute warps' export-band stores (ordered before this
          // thread by the named barrier) before the partial sums
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
          for (int j2 = 0; j2 < 3; ++j2) {
            unsigned long long u = (unsigned long long)__double_as_longlong(part[j2]);
            if (u == kSlotEmpty) u = 0x7ff8000000000000ull;
            st_relaxed_gpu_u64(&ring[c * 4 + j2], u);
          }
        }
        __syncwarp();
      };
      bool polled[NL];
      auto poll = [&](int L) {  // every CTA's slot of the lane's reduction -> PCG scalars in st[L]
        double v[3];
        const unsigned long long* const ring = lane_slots(L) + (size_t)(st[L].seq % 3) * gs * 4;
        constexpr int KS = (kMaxGroupCTAs + 31) / 32;
        unsigned long long u[KS][3];
#pragma unroll
        for (int t = 0; t < KS; ++t)
#pragma unroll
          for (int j2 = 0; j2 < 3; ++j2) u[t][j2] = lane + 32 * t < gs ? kSlotEmpty : 0ull;
        for (;;) {
          bool done = true;
#pragma unroll
          for (int t = 0; t < KS; ++t)
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2)
              if (u[t][j2] == kSlotEmpty) u[t][j2] = ld_relaxed_gpu_u64(&ring[(lane + 32 * t) * 4 + j2]);
#pragma unroll
          for (int t = 0; t < KS; ++t)
#pragma unroll
            for (int j2 = 0; j2 < 3; ++j2) done = done && u[t][j2] != kSlotEmpty;
          if (__all_sync(0xffffffffu, done)) break;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: the peers' export-band stores
#pragma unroll
        for (int j2 = 0; j2 < 3; ++j2) {
          double acc = 0.0;
#pragma unroll
          for (int t = 0; t < KS; ++t) acc += __longlong_as_double((long long)u[t][j2]);
          v[j2] = warp_allsum(acc);
        }
        // PCG scalars of iteration it (R28; R7 breakdowns)
        const int it = st[L].its + 1;
        const double sigma = v[0];
        if (lane == 0) {
          if (sigma == 0.0) {
            st[L].seq = st[L].seq + 1;
            st[L].live = 2;  // breakdown: prolong d as it stands
          } else {
            const double rho = st[L].rho;
            const double alpha = rho / sigma;
            const double rho_new = rho - 2.0 * alpha * v[1] + alpha * alpha * v[2];
            const bool stop = it >= m || !(rho_new > 0.0);
            st[L].alpha = alpha;
            st[L].beta = rho_new / rho;
            st[L].rho = rho_new;
            st[L].its = it;
            st[L].seq = st[L].seq + 1;
            st[L].live = stop ? 3 : 1;  // 3: last pass B, then prolong
          }
        }
        __syncwarp();
        polled[L] = true;
      };
      auto next_live = [&](int from) {  // first live lane after `from`, cyclic (from itself last)
        int r = -1;
#pragma unroll
        for (int k2 = NL; k2 >= 1; --k2) {
          const int L2 = (from + k2) % NL;
          if (live[L2]) r = L2;
        }
        return r;
      };
#pragma unroll
      for (int L = 0; L < NL; ++L) {
        polled[L] = false;
        if (live[L]) {
          take_part(L);
          publish(L);
        }
      }
      int R = next_live(NL - 1);
      bool delivered = false;
      while (R >= 0) {
        if (!delivered) {
          if (!polled[R]) poll(R);
          nbar_arrive(bar_res(R), NT);
        }
        delivered = false;
        polled[R] = false;
        if (st[R].live != 1) {  // the lane's last pass: no more partials from it
          live[R] = false;
          R = next_live(R);
          continue;
        }
        const int Rn = next_live(R);  // the result the compute warps need after PART(R)
        if (Rn != R && !polled[Rn]) poll(Rn);  // while they run R's passes
        take_part(R);
        if (Rn != R) {
          nbar_arrive(bar_res(Rn), NT);
          delivered = true;
        }
        publish(R);
        R = Rn;
      }
    } else {
      // ================= compute warps =================
      double q[NL][RPT];
      auto pass_a = [&](int L, int it) {
        const int rb = st[L].rb, nr = st[L].nr;
        const int4 band = st[L].band;
        const double* sp = lane_sp(L);
        const uint8_t* sdc = lane_id(L);
        const double* spv = lane_pv(L);
        const int32_t* spdl = lane_pdl(L);
        const double* spdg = lane_pdg(L);
        const double* spdi = lane_pdi(L);
        double v[3] = {0.0, 0.0, 0.0};
        // !PAT: SELL-Z entries of four rows (codes, 16-bit column offsets, slice bases)
        constexpr int W4 = W / 4 > 0 ? W / 4 : 1, W2 = W / 2 > 0 ? W / 2 : 1;
        uint32_t zc[4][W4], zd[4][W2];
        const int32_t* skb = lane_kb(L);
        auto zload = [&](int b) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = (4 * b + u) * NC + ct;
            if (i < nr) {
              const int64_t row = (int64_t)rb + i;
              if (W == 4) {
                zc[u][0] = __ldg(reinterpret_cast<const unsigned int*>(Lm.code) + row);
                const uint2 dd = __ldg(reinterpret_cast<const uint2*>(Lm.d16) + row);
                zd[u][0] = dd.x;
                zd[u][W2 - 1] = dd.y;
              } else {
                const uint2 cc = __ldg(reinterpret_cast<const uint2*>(Lm.code) + row);
                zc[u][0] = cc.x;
                zc[u][W4 - 1] = cc.y;
                const uint4 dd = __ldg(reinterpret_cast<const uint4*>(Lm.d16) + row);
                zd[u][0] = dd.x, zd[u][1] = dd.y, zd[u][2] = dd.z, zd[u][W2 - 1] = dd.w;
              }
            }
          }
        };
#pragma unroll
        for (int b = 0; b < RPT / 4; ++b) {
          if (!PAT) zload(b);  // this batch's entries (in flight with the TMEM load)
          double rr4[4];
          tm_ld4(tcol(L, 0, 4 * b), rr4);
          tm_ld_wait();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * b + u;
            const int i = j * NC + ct;
            if (i < nr) {
              const double pi = sp[i];
              const int pt = sdc[i];
              double off = 0.0, dg, di;
              if (PAT) {
#pragma unroll
                for (int k = 0; k < W; ++k) off += spv[pt * W + k] * sp[i + spdl[pt * W + k]];
                dg = spdg[pt];
                di = spdi[pt];
              } else {
                const int32_t* kb = skb + (i >> 5) * W;  // this row's slice bases (shared memory)
                bool wide = false;
#pragma unroll
                for (int k = 0; k < W; ++k) wide = wide || kb[k] < 0;
                if (!wide) {
#pragma unroll
                  for (int k = 0; k < W; ++k) {
                    const uint32_t code = (zc[u][k / 4] >> (8 * (k % 4))) & 0xffu;
                    const int li = kb[k] - rb + (int)((zd[u][k / 2] >> (16 * (k % 2))) & 0xffffu);
                    off += stab[code] * sp[li];
                  }
                } else {  // a slice with a wide group (int32 columns): generic decoder
                  off = r2_wide_row<W>(Lm, (int64_t)rb + i, stab, sp - rb);
                }
                dg = stab[pt];
                di = sinv[pt];
              }
              const double qi = __fma_rn(dg, pi, off);
              q[L][j] = qi;
              const double zi = __dmul_rn(di, rr4[u]);
              const double dq = __dmul_rn(di, qi);
              v[0] += pi * qi;
              v[1] += zi * qi;
              v[2] += qi * dq;
              if (i < band.x || i >= band.y) __stcg(&R2_PUB(pub_q, it & 1, rb)[i], qi);
            }
          }
        }
        // this warp's partials -> shared memory, then hand them to the reduction warp
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double s = warp_sum(v[j]);
          if (lane == 0) red[L][j][w - 1] = s;
        }
        nbar_arrive(bar_part(L), NT);
      };
#pragma unroll
      for (int L = 0; L < NL; ++L)
        if (live[L]) pass_a(L, 1);
      for (;;) {
        bool any = false;
#pragma unroll
        for (int L = 0; L < NL; ++L) {
          if (!live[L]) continue;
          any = true;
          nbar_sync(bar_res(L), NT);  // the reduction warp's scalars of this iteration
          const int phase = st[L].live;
          const int it = st[L].its;    // the iteration just reduced (unchanged on breakdown)
          const double alpha = st[L].alpha, beta = st[L].beta;
          const int rb = st[L].rb, nr = st[L].nr;
          const int4 band = st[L].band;
          double* sp = lane_sp(L);
          const uint8_t* sdc = lane_id(L);
          const double* spdi = lane_pdi(L);
          if (phase != 2) {
            const bool stop = phase == 3;
            // ghost rows of p_{it+1} (R29): the neighbours' published q_it and r_{it-1}
            // are copied into the staging buffer asynchronously (cp.async, no
            // registers) while pass B runs; p_it of a ghost row is already in sp
            // (bitwise the owner's value).  The L1 lines of the published arrays were
            // invalidated by the reduction warp's acquire fence (CCTL.IVALL).
            const int ng = band.z + band.w;
            auto ghost_row = [&](int t) { return t < band.z ? t - band.z : nr + (t - band.z); };
            if (!stop) {
              for (int t = ct; t < ng; t += NC) {
                const int li = ghost_row(t);
                cp_async8(&sstage[t], &R2_PUB(pub_q, it & 1, rb)[li]);
                cp_async8(&sstage[gmax + t], &R2_PUB(pub_r, (it - 1) & 1, rb)[li]);
              }
              cp_async_commit();
            }
            // pass B: d += alpha p, r -= alpha q, p_{it+1} = D^-1 r + beta p (own rows)
#pragma unroll
            for (int b = 0; b < RPT / 4; ++b) {
              double dd[4], rr[4];
              if (it > 1) tm_ld4(tcol(L, 1, 4 * b), dd);
              tm_ld4(tcol(L, 0, 4 * b), rr);
              tm_ld_wait();
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = 4 * b + u;
                const int i = j * NC + ct;
                if (it == 1) dd[u] = 0.0;
                if (i < nr) {
                  const double pi = sp[i];
                  dd[u] = it == 1 ? alpha * pi : __fma_rn(alpha, pi, dd[u]);
                  if (!stop) {
                    const double rn = __fma_rn(-alpha, q[L][j], rr[u]);
                    rr[u] = rn;
                    const double pn = __fma_rn(beta, pi, __dmul_rn(PAT ? spdi[sdc[i]] : sinv[sdc[i]], rn));
                    sp[i] = pn;
                    if (i < band.x || i >= band.y) {
                      __stcg(&R2_PUB(pub_r, it & 1, rb)[i], rn);
                      __stcg(&R2_PUB(pub_p, (it + 1) & 1, rb)[i], pn);
                    }
                  }
                }
              }
              tm_st4(tcol(L, 1, 4 * b), dd);
              tm_st4(tcol(L, 0, 4 * b), rr);
            }
            if (!stop) {
              cp_async_wait_all();  // this thread's own copies
              for (int t = ct; t < ng; t += NC) {
                const int li = ghost_row(t);
                sp[li] = __fma_rn(beta, sp[li],
                                  __dmul_rn(sinv[__ldg(&D.code[rb + li])], __fma_rn(-alpha, sstage[t], sstage[gmax + t])));
              }
            }
            tm_st_wait();
          }
          if (phase != 1) {
            // a4: restricted prolongation of the chunk's owned rows (d of the rows this thread owns)
            if (it > 0) {
#pragma unroll
              for (int b = 0; b < RPT / 4; ++b) {
                double dd[4];
                tm_ld4(tcol(L, 1, 4 * b), dd);
                tm_ld_wait();
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int i = (4 * b + u) * NC + ct;
                  if (i < nr) {
                    const int32_t s = __ldg(&own_slot[rb + i]);
                    if (s >= 0) x[s] = x[s] + dd[u];
                  }
                }
              }
            }
            if (ct == 0 && c == 0) {
              const int lp = st[L].lp;
              S.its[lp] = it;
              S.inner_total[lp] += it;
              S.active[lp] = 0;
            }
            live[L] = false;
            continue;
          }
          nbar_sync(kBarCompute, NC);  // p_{it+1} (own rows + ghosts) complete before the gathers
          pass_a(L, it + 1);
        }
        if (!any) break;
      }
    }
    __syncthreads();  // both roles finished the pair (lane state and shared memory reused next)
  }
#undef R2_PUB
  // ---- release TMEM ----
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tbase));
}

}  // namespace ras
