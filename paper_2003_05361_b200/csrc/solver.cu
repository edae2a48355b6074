// C ABI: ras_setup / ras_solve (sync mode) / ras_stats / ras_free.
// PAPER Alg. 1 (P233-245): initialization_and_setup, then the solve loop
// {local solve; exchange; update boundary; check convergence}; gather.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "ctx.h"
#include "kernels.cuh"
#include "resident2.cuh"
#include "plan_internal.h"
#include "ras.h"
#include "ras_plan.h"

namespace ras {

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

ras_status set_err(ras_ctx* c, ras_status s, const std::string& m) {
  if (c)
    c->err = m;
  else
    set_tls_error(m);
  return s;
}

ras_status cuda_err(ras_ctx* c, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_err(c, e == cudaErrorMemoryAllocation ? RAS_ENOMEM : RAS_ECUDA, m);
}

void* dalloc(ras_ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 8;
  bytes = (bytes + 255) / 256 * 256;
  void* p = nullptr;
  if (c->dev_alloc) {
    p = c->dev_alloc(bytes, c->alloc_user);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
  }
  if (p) c->bufs.push_back(DevBuf{p, bytes, false});
  return p;
}

// Always cudaMalloc (a base allocation that can be exported as a CUDA IPC
// window to the peer GPUs: x storage and the detector board).
// Raise a kernel's dynamic shared-memory cap to everything the device allows.
// The attribute is per function and process-wide: setting it to the launch's own
// size would race between contexts (e.g. loopback ranks on host threads) that
// launch the same kernel with different sizes; the device maximum never shrinks.
ras_status allow_smem(ras_ctx* c, const void* fn) {
  int optin = 0;
  RAS_CUDA(c, cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  cudaFuncAttributes fa{};
  RAS_CUDA(c, cudaFuncGetAttributes(&fa, fn));
  RAS_CUDA(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
  return RAS_OK;
}

void dfree(ras_ctx* c, void* p) {
  for (size_t i = 0; i < c->bufs.size(); ++i)
    if (c->bufs[i].ptr == p) {
      if (c->dev_free && !c->bufs[i].raw)
        c->dev_free(p, c->alloc_user);
      else
        cudaFree(p);
      c->bufs.erase(c->bufs.begin() + i);
      return;
    }
}

void* dalloc_raw(ras_ctx* c, size_t bytes) {
  bytes = std::max<size_t>(256, (bytes + 255) / 256 * 256);
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  if (cudaMemsetAsync(p, 0, bytes, c->stream) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  c->bufs.push_back(DevBuf{p, bytes, true});
  return p;
}


// Multi-rank exchange of halo requests over NCCL (setup only): every rank
// learns which of its owned values each peer needs, in the peer's halo order.
static ras_status exchange_requests(ras_ctx* c) {
  ras_plan* pl = c->plan;
  const int W = c->world, me = c->rank;
  std::vector<int64_t> my_counts(W);
  for (int r = 0; r < W; ++r) my_counts[r] = pl->halo_off[r + 1] - pl->halo_off[r];
  int64_t *d_counts = nullptr, *d_all = nullptr;
  TRY(upload(c, &d_counts, my_counts));
  TRY(zalloc(c, &d_all, (size_t)W * W));
  TRY(coll_allgather(c, d_counts, d_all, W, ncclInt64, c->stream));
  std::vector<int64_t> all((size_t)W * W);
  RAS_CUDA(c, cudaMemcpyAsync(all.data(), d_all, all.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  // all[q*W + r] = how many values rank q needs from rank r
  int64_t tot_in = 0;
  for (int q = 0; q < W; ++q) tot_in += all[(size_t)q * W + me];
  int64_t *d_req = nullptr, *d_inc = nullptr;
  TRY(upload(c, &d_req, pl->halo_gid, 1));
  TRY(zalloc(c, &d_inc, std::max<int64_t>(tot_in, 1)));
  std::vector<int64_t> inc_off(W + 1, 0);
  for (int q = 0; q < W; ++q) inc_off[q + 1] = inc_off[q] + all[(size_t)q * W + me];
  std::vector<Xfer> snd, rcv;
  for (int r = 0; r < W; ++r) {
    if (r == me) continue;
    const int64_t cnt = pl->halo_off[r + 1] - pl->halo_off[r];
    if (cnt) snd.push_back(Xfer{r, d_req + pl->halo_off[r], (size_t)cnt});
    const int64_t inc = all[(size_t)r * W + me];
    if (inc) rcv.push_back(Xfer{r, d_inc + inc_off[r], (size_t)inc});
  }
  TRY(coll_sendrecv(c, snd, rcv, ncclInt64, c->stream));
  std::vector<int64_t> inc(std::max<int64_t>(tot_in, 1));
  RAS_CUDA(c, cudaMemcpyAsync(inc.data(), d_inc, inc.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int q = 0; q < W; ++q) {
    if (q == me) continue;
    // where my segment lands in q's halo: sum of what q needs from ranks < me
    int64_t roff = 0;
    for (int r = 0; r < me; ++r) roff += all[(size_t)q * W + r];
    const int64_t cnt = all[(size_t)q * W + me];
    ras_status s = ras_plan_set_send(pl, q, cnt, inc.data() + inc_off[q], roff);
    if (s != RAS_OK) return set_err(c, s, tls_error());
  }
  return RAS_OK;
}

static void compute_model_bytes(ras_ctx* c) {
  const ras_plan* pl = c->plan;
  const double rows = (double)pl->rows_local;
  int64_t owned = pl->n_own;
  const double nnz_off = (double)(pl->nnz_local - pl->rows_local);
  // compulsory bytes, real (unpadded) rows and entries.  Plain
  // SELL: 8 B value + 4 B column per entry, 8 B diagonal; SELL-Z: 1 B code +
  // 2 B column offset (+ 4 B base per 32 entries), 1 B diagonal code.
  // SELL-Z is lane-packed to the padded width: every row moves Wp entries.
  const double eb = c->z ? (1.0 + 2.0 + 4.0 / 32.0) : 12.0;
  const double db = c->z ? 1.0 : 8.0;
  const double ent_R = c->z ? rows * pl->zR_w : (double)pl->nnz_residual;
  const double ent_L = c->z ? rows * pl->zL_w : nnz_off;
  c->mb.residual = rows * (8 /*b*/ + db /*diag*/ + 4 /*own_slot*/ + 8 /*x*/ + 8 /*r*/ + 8 /*p*/) + ent_R * eb;
  if (c->fuse_p) {
    // pass 1 with the fused p update: r (or z), diag, p_old in; p_new, q out (+ off-diagonal entries)
    c->mb.spmv_dot = rows * (8 /*r|z*/ + 8 /*diag*/ + 8 /*p_old*/ + 8 /*p_new*/ + 8 /*q*/) + nnz_off * 12.0;
    c->mb.pupdate = 0.0;
  } else {
    c->mb.spmv_dot = rows * (8 /*p*/ + db /*diag*/ + 8 /*q*/) + ent_L * eb;
    c->mb.pupdate = rows * (db /*diag*/ + 8 /*r*/ + 16 /*p*/);
  }
  c->mb.update_dot = rows * (8 /*p*/ + 8 /*q*/ + db /*diag*/ + 16 /*r*/ + 16 /*d*/);
  c->mb.prolong = rows * 4.0 + (double)owned * (8 /*d*/ + 16 /*x*/);
  c->mb.pack = (double)c->n_send * (4 + 8 + 8);
  // BLOCK / RESIDENT: one launch = the whole local solve of every subdomain; its
  // compulsory HBM traffic is r, p (from k_residual), the local matrix and
  // diagonal once, the prolong map, and x[S_p] read + written.  Every further
  // PCG iteration runs from shared memory / registers / L2.
  c->mb.local_solve = rows * (8 /*r*/ + 8 /*p*/ + db /*diag*/ + 4 /*own_slot*/) + ent_L * eb + (double)owned * 16.0;
}

// RESIDENT path setup (k_resident_pcg): group count / size, rows per thread,
// export bands, barrier counters and partial-sum slots.  Leaves c->path alone
// when no configuration fits (the caller falls back to TILED).
static const void* resident_kernel(int rpt, bool z, int w, bool tol, bool pat) {
#define RAS_RK3(RPT, W, Z, PAT) \
  return tol ? (const void*)k_resident_pcg<RPT, W, Z, true, PAT> : (const void*)k_resident_pcg<RPT, W, Z, false, PAT>;
#define RAS_RK2(RPT, W)     \
  if (pat) {                \
    RAS_RK3(RPT, W, true, true) \
  } else {                  \
    RAS_RK3(RPT, W, true, false) \
  }
#define RAS_RK(RPT)                     \
  if (z) {                              \
    if (w == 4) {                       \
      RAS_RK2(RPT, 4)                   \
    } else {                            \
      RAS_RK2(RPT, 8)                   \
    }                                   \
  } else {                              \
    RAS_RK3(RPT, 0, false, false)       \
  }
  // instantiated rows-per-thread counts: 4, 8 and kResidMaxRPT (the register budget's limit)
  if (rpt <= 4) {
    RAS_RK(4)
  } else if (rpt <= 8) {
    RAS_RK(8)
  } else {
    RAS_RK(kResidMaxRPT)
  }
#undef RAS_RK3
#undef RAS_RK2
#undef RAS_RK
}

// k_resident2 instantiations: rows per thread x SELL-Z width (4 / 8) x lanes x row-pattern SpMV
template <int RPT, int NL, bool PAT>
static const void* r2_fn(int w) {
  return w == 4 ? (const void*)k_resident2<RPT, 4, NL, PAT> : (const void*)k_resident2<RPT, 8, NL, PAT>;
}
template <int RPT, bool PAT>
static const void* r2_fn_l(int w, int lanes) {
  if constexpr (RPT <= 16) {
    if (lanes == 2) return r2_fn<RPT, 2, PAT>(w);
  }
  return lanes == 1 ? r2_fn<RPT, 1, PAT>(w) : nullptr;
}
template <bool PAT>
static const void* resident2_kernel_p(int rpt, int w, int lanes) {
  if (rpt <= 4) return r2_fn_l<4, PAT>(w, lanes);
  if (rpt <= 8) return r2_fn_l<8, PAT>(w, lanes);
  if (rpt <= 12) return r2_fn_l<12, PAT>(w, lanes);
  if (rpt <= 16) return r2_fn_l<16, PAT>(w, lanes);
  return r2_fn_l<kR2MaxRPT, PAT>(w, lanes);
}
static const void* resident2_kernel(int rpt, int w, int lanes, bool pat) {
  return pat ? resident2_kernel_p<true>(rpt, w, lanes) : resident2_kernel_p<false>(rpt, w, lanes);
}

// Per-chunk export bands / ghost zones and (PAT) row-pattern tables of every
// local subdomain for a group of gs CTAs (chunk = the rows of one CTA).
struct ResidLayout {
  std::vector<int4> band;
  int glo_max = 0, ghi_max = 0;
  bool pat = false;
  std::vector<int32_t> pat_off, pat_cnt, pat_dlt;
  std::vector<double> pat_val, pat_diag;
  std::vector<uint8_t> pid;
};

static int chunk_rows(int n, int gs) { return ((n / 32 + gs - 1) / gs) * 32; }

static void resident_layout(const ras_ctx* c, int gs, bool want_pat, ResidLayout& Lo) {
  const ras_plan* pl = c->plan;
  const int nl = c->nl;
  Lo.band.assign((size_t)nl * gs, make_int4(0, 0, 0, 0));
  Lo.glo_max = Lo.ghi_max = 0;
  for (int lp = 0; lp < nl; ++lp) {
    const auto& S = pl->subs[lp];
    const int n = (int)S.nrows_pad, ch = chunk_rows(n, gs);
    std::vector<int> lo(gs, 0), hi(gs), len(gs), glo(gs, 0), ghi(gs, 0);
    for (int cc = 0; cc < gs; ++cc) {
      const int a = std::min(n, cc * ch);
      len[cc] = std::min(n, a + ch) - a;
      hi[cc] = len[cc];
    }
    for (int i = 0; i < n; ++i) {
      const int ci = i / ch;
      for (int64_t e = pl->Ap_ptr[S.row_off + i]; e < pl->Ap_ptr[S.row_off + i + 1]; ++e) {
        const int j = pl->Ap_col[e], cj = j / ch;
        if (cj == ci) continue;
        const int lj = j - cj * ch;
        if (lj < len[cj] / 2)
          lo[cj] = std::max(lo[cj], lj + 1);
        else
          hi[cj] = std::min(hi[cj], lj);
        const int li = j - ci * ch;  // column relative to the reading chunk
        if (li < 0)
          glo[ci] = std::max(glo[ci], -li);
        else
          ghi[ci] = std::max(ghi[ci], li - len[ci] + 1);
      }
    }
    for (int cc = 0; cc < gs; ++cc) {
      Lo.band[(size_t)lp * gs + cc] = make_int4(lo[cc], hi[cc], glo[cc], ghi[cc]);
      Lo.glo_max = std::max(Lo.glo_max, glo[cc]);
      Lo.ghi_max = std::max(Lo.ghi_max, ghi[cc]);
    }
  }
  // row-pattern dictionary per chunk (PAT): SELL-Z matrices whose every chunk has
  // <= kMaxPat distinct rows (diagonal + (delta, value) list); then no matrix
  // stream from L2 in the SpMV
  Lo.pat_off.assign((size_t)nl * gs, 0);
  Lo.pat_cnt.assign((size_t)nl * gs, 0);
  Lo.pat_dlt.clear();
  Lo.pat_val.clear();
  Lo.pat_diag.clear();
  Lo.pid.clear();
  bool pat = want_pat && c->z;
  if (pat) {
    const int W = c->zwL;
    Lo.pid.assign((size_t)c->rows_pad, 0);
    std::vector<uint64_t> key;
    for (int lp = 0; lp < nl && pat; ++lp) {
      const auto& S = pl->subs[lp];
      const int n = (int)S.nrows_pad, ch = chunk_rows(n, gs);
      for (int cc = 0; cc < gs && pat; ++cc) {
        const int a = std::min(n, cc * ch), e = std::min(n, a + ch);
        std::vector<std::vector<uint64_t>> keys;  // this chunk's distinct patterns
        Lo.pat_off[(size_t)lp * gs + cc] = (int32_t)Lo.pat_diag.size();
        for (int i = a; i < e; ++i) {
          const int64_t row = S.row_off + i;
          key.assign(1 + 2 * W, 0);
          double dg = pl->diag[row];
          std::memcpy(&key[0], &dg, 8);
          int k = 0;
          for (int64_t q = pl->Ap_ptr[row]; q < pl->Ap_ptr[row + 1]; ++q) {
            const int j = pl->Ap_col[q];
            if (j == i) continue;
            if (k == W) {
              pat = false;
              break;
            }
            const double v = pl->Ap_val[q];
            key[1 + k] = (uint64_t)(uint32_t)(j - i);
            std::memcpy(&key[1 + W + k], &v, 8);
            ++k;
          }
          if (!pat) break;
          size_t id = 0;
          while (id < keys.size() && keys[id] != key) ++id;
          if (id == keys.size()) {
            if (keys.size() == (size_t)kMaxPat) {
              pat = false;
              break;
            }
            keys.push_back(key);
            Lo.pat_diag.push_back(dg);
            for (int t = 0; t < W; ++t) {
              Lo.pat_dlt.push_back((int32_t)(uint32_t)key[1 + t]);
              double v;
              std::memcpy(&v, &key[1 + W + t], 8);
              Lo.pat_val.push_back(v);
            }
          }
          Lo.pid[(size_t)row] = (uint8_t)id;
        }
        Lo.pat_cnt[(size_t)lp * gs + cc] = (int32_t)keys.size();
      }
    }
  }
  Lo.pat = pat;
}

// RESIDENT path setup: group count / size, kernel version and rows per thread,
// export bands, barrier counters and partial-sum slots.  Leaves c->path alone
// when no configuration fits (the caller falls back to TILED).
//   v2 (k_resident2, r and d in tensor memory): fixed-m solves on row-pattern
//      matrices; NL = 2 interleaved subdomains when two lanes fit a CTA, else
//      NL = 1 with chunks up to kR2MaxRPT x 768 rows;
//   v1 (k_resident_pcg): everything else that fits (tolerance solves, SELL-Z
//      stream / plain SELL matrices).  RAS_RESIDENT_KERNEL=1 forces v1 (A/B runs).
static ras_status setup_resident(ras_ctx* c, int nmax) {
  int sms = 0, smem_optin = 0;
  RAS_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  RAS_CUDA(c, cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  const int nl = c->nl;
  const bool tol = c->opt.local_solver == RAS_LS_EXACT_PCG || c->opt.inner_tol > 0.0;
  const char* env = getenv("RAS_RESIDENT_KERNEL");
  const bool v2_ok = c->z && !tol && !(env && env[0] == '1');
  // fewest groups with the largest concurrency that fits `cap` rows per CTA
  auto pick = [&](int units, int cap, int* k_out, int* gs_out) {
    int kfit = 0;
    for (int k = 1; k <= std::min(units, sms); ++k)
      if (chunk_rows(nmax, std::min(sms / k, kMaxGroupCTAs)) <= cap) kfit = k;
    if (kfit == 0) return false;
    const int waves = (units + kfit - 1) / kfit;
    int k = kfit;
    while (k > 1 && (units + k - 2) / (k - 1) == waves) --k;
    *k_out = k;
    *gs_out = std::min(sms / k, kMaxGroupCTAs);
    return true;
  };
  ResidLayout Lo;
  int k = 0, gs = 0, chunk = 0, lanes = 0;
  size_t smem = 0;
  const size_t r2_static = 8 * (2 * 3 * (kNC_R2 / 32) + 256) + sizeof(R2Lane) * 2 + 64;
  if (v2_ok) {
    for (int NL = 2; NL >= 1 && !lanes; --NL) {
      const int maxrpt = std::min(kR2ColBlk / 4 / NL, kR2MaxRPT);
      if (!pick((nl + NL - 1) / NL, maxrpt * kNC_R2, &k, &gs)) continue;
      chunk = chunk_rows(nmax, gs);
      resident_layout(c, gs, true, Lo);  // row patterns if every chunk has <= kMaxPat, else the SELL-Z stream
      // NL lanes + the ghost staging buffer (q, r of the widest ghost zones)
      const size_t dyn = (size_t)NL * 8 * r2_lane_words(Lo.glo_max, chunk, Lo.ghi_max, c->zwL, Lo.pat) +
                         (size_t)16 * (Lo.glo_max + Lo.ghi_max);
      if (dyn + r2_static + 1024 <= (size_t)smem_optin) {
        lanes = NL;
        smem = dyn;
      }
    }
  }
  if (!lanes) {
    // v1: shared memory per chunk row p, r, d (24 B) + diagonal (SELL-Z: 1 B code, plain: 8 B)
    const int row_b = c->z ? 25 : 32;
    const int cap = std::min(kResidMaxRPT * kNT_RESID, ((smem_optin - 4096 - 2048) / row_b) / 32 * 32);
    if (!pick(nl, cap, &k, &gs)) return RAS_OK;
    chunk = chunk_rows(nmax, gs);
    if (chunk > cap) return RAS_OK;
#ifdef RAS_NO_PAT  // timing experiment: force the SELL-Z stream
    resident_layout(c, gs, false, Lo);
#else
    resident_layout(c, gs, true, Lo);
#endif
    const size_t pat_smem = Lo.pat ? (size_t)kMaxPat * (8 * (size_t)c->zwL + 8 + 8 + 4 * (size_t)c->zwL) + 8 : 0;
    smem = (size_t)8 * (Lo.glo_max + Lo.ghi_max) + (size_t)24 * chunk +
           (c->z ? 4096 + (size_t)((chunk + 7) & ~7) : (size_t)8 * chunk) + pat_smem;
    if (smem + 2048 > (size_t)smem_optin) return RAS_OK;  // ghost zones too wide: TILED
  }
  const int nt = lanes ? kNT_R2 : kNT_RESID;
  const int ntr = lanes ? kNC_R2 : kNT_RESID;  // threads that own rows
  const int need = (chunk + ntr - 1) / ntr;
  int rpt;
  if (lanes) {
    rpt = need <= 4 ? 4 : need <= 8 ? 8 : need <= 12 ? 12 : need <= 16 ? 16 : kR2MaxRPT;
    if (lanes == 2 && rpt > 16) return set_err(c, RAS_ESTATE, "resident v2: two lanes need <= 16 rows per thread");
  } else {
    rpt = need <= 4 ? 4 : need <= 8 ? 8 : kResidMaxRPT;
  }
  const void* fn = lanes ? resident2_kernel(rpt, c->zwL, lanes, Lo.pat)
                         : resident_kernel(rpt, c->z, c->z ? c->zwL : c->wL, tol, Lo.pat);
  if (!fn) return RAS_OK;
  TRY(allow_smem(c, fn));
  int per_sm = 0;
  RAS_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, smem));
  if (per_sm < 1) return RAS_OK;
  int4* dband;
  TRY(upload(c, &dband, Lo.band));
  c->resid_glo = Lo.glo_max;
  c->resid_ghi = Lo.ghi_max;
  // slot rings: one per (group, lane)
  TRY(zalloc(c, &c->d_resid_slots, (size_t)k * std::max(lanes, 1) * 3 * kResidNV * gs));
  double* q2;
  TRY(zalloc(c, &q2, (size_t)c->rows_pad));
  // published export-band values (kernels.cuh): pub_p[1] = k_residual's p, pub_r[0] = its r
  int32_t *dpo = nullptr, *dpc = nullptr, *dpd = nullptr;
  double *dpv = nullptr, *dpg = nullptr;
  uint8_t* dpid = nullptr;
  if (Lo.pat) {
    TRY(upload(c, &dpo, Lo.pat_off));
    TRY(upload(c, &dpc, Lo.pat_cnt));
    TRY(upload(c, &dpd, Lo.pat_dlt, 1));
    TRY(upload(c, &dpv, Lo.pat_val, 1));
    TRY(upload(c, &dpg, Lo.pat_diag, 1));
    TRY(upload(c, &dpid, Lo.pid, 1));
  }
  c->resid_pat = Lo.pat;
  c->resid_lanes = lanes;
  c->RC = ResidentCtl{dband, c->d_resid_slots, dpo, dpc, dpv, dpd, dpg, dpid,
                      {c->d_p2, c->d_p}, {c->d_r, c->d_d}, {c->d_q, q2}, k, gs};
  c->resid_rpt = rpt;
  c->resid_chunk = chunk;
  c->resid_smem = smem;
  c->path = RAS_PCG_RESIDENT;
  return RAS_OK;
}

// a3' setup: IC(0)/ILU(0) factors + level sets on the host (factor.cpp), uploaded once
static ras_status upload_tri(ras_ctx* c, const TriHost& H, TriBuf& B) {
  const ras_plan* pl = c->plan;
  int32_t *rows, *rp, *col, *bat, *slo, *lnc;
  double *val, *diag;
  int4* ch;
  TRY(upload(c, &rows, H.rows, 1));
  TRY(upload(c, &rp, H.rp, 1));
  TRY(upload(c, &col, H.col, 1));
  TRY(upload(c, &val, H.val, 1));
  TRY(upload(c, &diag, H.diag, 1));
  std::vector<int4> chunks(H.chunk.size());
  for (size_t i = 0; i < chunks.size(); ++i)
    chunks[i] = make_int4(H.chunk[i][0], H.chunk[i][1], H.chunk[i][2], H.chunk[i][3]);
  TRY(upload(c, &ch, chunks, 1));
  TRY(upload(c, &bat, H.batched, 1));
  TRY(upload(c, &slo, H.sub_lev_off, 1));
  TRY(upload(c, &lnc, H.lev_nchunks, 1));
  B.dev = TriDev{rows, rp, col, val, diag, ch, bat, slo, lnc};
  B.nchunks = (int32_t)H.chunk.size();
  B.nlev_slots = (int32_t)H.lev_nchunks.size();
  B.sub_lev_off = H.sub_lev_off;
  B.sub_nlev = H.sub_nlev;
  B.sub_c0 = H.sub_chunk_begin;
  B.sub_nc.resize(H.sub_chunk_begin.size());
  for (size_t i = 0; i < B.sub_nc.size(); ++i) B.sub_nc[i] = H.sub_chunk_end[i] - H.sub_chunk_begin[i];
  TRY(zalloc(c, &B.d_lev_done, (size_t)std::max(B.nlev_slots, 1)));
  B.sub_max_lev = H.sub_max_lev;
  B.cl_ok = H.max_deps <= 4 && H.max_levels < kTrcLevSmem;  // k_trsv_cl: <= 4 deps / row, levels staged in smem
  if (B.cl_ok) {  // k_trsv_cl: the factor re-laid out by level-ordered position
    const size_t np = H.rows.size();
    std::vector<double> pdiv(np), pval(4 * np, 0.0);
    std::vector<int4> pcol(np);
    for (size_t k = 0; k < np; ++k) {
      pdiv[k] = H.diag[H.rows[k]];
      int32_t cc[4] = {-1, -1, -1, -1};
      for (int32_t e = H.rp[k], q = 0; e < H.rp[k + 1]; ++e, ++q) {
        cc[q] = H.col[e];
        pval[4 * k + q] = H.val[e];
      }
      pcol[k] = make_int4(cc[0], cc[1], cc[2], cc[3]);
    }
    int32_t *lp, *spo, *snl;
    double *dv, *pv;
    int4* pc;
    TRY(upload(c, &lp, H.lev_pos, 1));
    TRY(upload(c, &spo, H.sub_pos_off, 1));
    TRY(upload(c, &snl, H.sub_nlev, 1));
    TRY(upload(c, &dv, pdiv, 1));
    TRY(upload(c, &pc, pcol, 1));
    TRY(upload(c, &pv, pval, 2));
    B.cl = TriCl{lp, spo, snl, rows, dv, pc, (const double2*)pv};
    // k_trsv_pf: the chunks each chunk's rows depend on (chunk ids are in
    // position = level order, so the range covers earlier chunks only)
    std::vector<int32_t> pos_of_row((size_t)c->rows_pad, -1), chunk_of(np, 0);
    for (size_t k = 0; k < np; ++k) pos_of_row[H.rows[k]] = (int32_t)k;
    for (size_t cc = 0; cc < H.chunk.size(); ++cc)
      for (int32_t k = H.chunk[cc][0]; k < H.chunk[cc][1]; ++k) chunk_of[k] = (int32_t)cc;
    std::vector<int2> cdep(H.chunk.size(), make_int2(0, -1));
    for (size_t cc = 0; cc < H.chunk.size(); ++cc) {
      int32_t lo = INT32_MAX, hi = -1;
      for (int32_t k = H.chunk[cc][0]; k < H.chunk[cc][1]; ++k)
        for (int32_t e = H.rp[k]; e < H.rp[k + 1]; ++e) {
          const int32_t d = chunk_of[pos_of_row[H.col[e]]];
          lo = std::min(lo, d);
          hi = std::max(hi, d);
        }
      if (hi >= 0) cdep[cc] = make_int2(lo, hi);
    }
    TRY(upload(c, &B.d_cdep, cdep, 1));
    TRY(zalloc(c, &B.d_cflag, std::max<size_t>(H.chunk.size(), 1)));
  }
  // algorithmic bytes of one solve: per real row rows/rp/in/out/diag, per entry val+col
  B.bytes = (double)pl->rows_local * (4 + 4 + 8 + 8 + 8) + (double)(pl->nnz_local - pl->rows_local) / 2.0 * 12.0;
  return RAS_OK;
}

// k_trsv_ds routing tables of one factor for cluster size ncl (DSMEM-routed
// solve, kernels.cuh): false if the factor does not qualify (a dependency outside
// the previous level, > 4 dependencies or consumers, a level wider than
// kTrdRows rows per thread of the cluster)
static bool build_ds(ras_ctx* c, const TriHost& H, int ncl, TriBuf& B, ras_status* st) {
  *st = RAS_OK;
  const size_t np = H.rows.size();
  const int nl = (int)H.sub_nlev.size();
  std::vector<int32_t> pos_of_row((size_t)c->rows_pad, -1), lev_of(np, -1), cta_of(np, 0), prow(np), rb_off(nl + 1, 0),
      rbytes;
  std::vector<int4> psend(np, make_int4(-1, -1, -1, -1));
  for (size_t k = 0; k < np; ++k) {
    if (H.rows[k] >= (1 << 29)) return false;
    pos_of_row[H.rows[k]] = (int32_t)k;
  }
  for (int lp = 0; lp < nl; ++lp) {
    const int32_t* lev = H.lev_pos.data() + H.sub_pos_off[lp];
    const int nlev = H.sub_nlev[lp];
    rb_off[lp] = (int32_t)rbytes.size();
    rbytes.resize(rbytes.size() + (size_t)nlev * ncl, 0);
    for (int l = 0; l < nlev; ++l) {
      const int32_t b = lev[l], n = lev[l + 1] - b, q = (n + ncl - 1) / ncl;
      for (int32_t k = b; k < lev[l + 1]; ++k) {
        lev_of[k] = l;
        cta_of[k] = (k - b) / q;
      }
    }
    for (int l = 0; l < nlev; ++l) {
      const int32_t b = lev[l], n = lev[l + 1] - b, q = (n + ncl - 1) / ncl;
      if (q > kTrdRows * kNT_TRD) return false;
      for (int32_t k = b; k < lev[l + 1]; ++k) {
        const int32_t r = (k - b) / q, j = (k - b) % q, nd = H.rp[k + 1] - H.rp[k];
        if (nd > 4) return false;
        prow[k] = H.rows[k] | (nd << 29);
        for (int32_t qd = 0; qd < nd; ++qd) {
          const int32_t d = pos_of_row[H.col[H.rp[k] + qd]];
          if (d < 0 || lev_of[d] != l - 1) return false;
          // only values from other CTAs arrive through the mbarrier (DSMEM);
          // a CTA's own consumers are written with plain shared-memory stores
          if (cta_of[d] != r) rbytes[rb_off[lp] + (size_t)l * ncl + r] += 8;
          int32_t* sd = &psend[d].x;
          int w = 0;
          while (w < 4 && sd[w] >= 0) ++w;
          if (w == 4) return false;
          sd[w] = (r << 16) | (j * 4 + qd);
        }
      }
    }
  }
  rb_off[nl] = (int32_t)rbytes.size();
  std::vector<double> pdiv(np), pval(4 * np, 0.0);
  for (size_t k = 0; k < np; ++k) {
    pdiv[k] = H.diag[H.rows[k]];
    for (int32_t e = H.rp[k], qd = 0; e < H.rp[k + 1]; ++e, ++qd) pval[4 * k + qd] = H.val[e];
  }
  int32_t *dlp, *dspo, *dsnl, *drbo, *drb, *dpr;
  double *ddv, *dpv;
  int4* dps;
  if ((*st = upload(c, &dlp, H.lev_pos, 1)) || (*st = upload(c, &dspo, H.sub_pos_off, 1)) ||
      (*st = upload(c, &dsnl, H.sub_nlev, 1)) || (*st = upload(c, &drbo, rb_off, 1)) || (*st = upload(c, &drb, rbytes, 1)) ||
      (*st = upload(c, &dpr, prow, 1)) || (*st = upload(c, &ddv, pdiv, 1)) || (*st = upload(c, &dpv, pval, 2)) ||
      (*st = upload(c, &dps, psend, 1)))
    return false;
  B.ds = TriDs{dlp, dspo, dsnl, drbo, drb, dpr, ddv, (const double2*)dpv, dps};
  B.ds_ok = true;
  B.ds_ncl = ncl;
  return true;
}

static int trsv_ds_fit(ras_ctx* c, int k) {  // co-resident k_trsv_ds clusters of k CTAs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)k);
  cfg.blockDim = dim3(kNT_TRD);
  cfg.dynamicSmemBytes = (size_t)2 * kTrdSlots * sizeof(double);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)k;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_trsv_ds, &cfg) != cudaSuccess) n = 0;
  cudaGetLastError();
  if (getenv("RAS_TRSV_DEBUG")) fprintf(stderr, "k_trsv_ds: %d co-resident clusters of %d CTAs\n", n, k);
  return n;
}

static ras_status upload_factors(ras_ctx* c) {
  TriHost F, B;
  try {
    build_factors(c->plan, c->opt.local_solver, F, B);
  } catch (const Fail& f) {
    return set_err(c, f.st, f.msg);
  }
  TRY(upload_tri(c, F, c->tri_f));
  TRY(upload_tri(c, B, c->tri_b));
  TRY(zalloc(c, &c->d_z, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_y, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_trsv_ctr, (size_t)2 * (c->nl + 1)));
  {
    // A/B knob: "sf" = the sync-free kernel (measured 2x slower than the level
    // barriers on B200: profiles/r02_trsv.md), default the level-barrier kernel
    const char* e = getenv("RAS_TRSV");
    c->trsv_sf = e && std::strcmp(e, "sf") == 0;
    c->trsv_mode = c->trsv_sf ? 2 : (e && std::strcmp(e, "level") == 0) ? 1 : (e && std::strcmp(e, "pf") == 0) ? 3 : 0;
  }
  if (c->trsv_mode == 0 && c->tri_f.cl_ok && c->tri_b.cl_ok) {
    // cluster-resident solve: 16-CTA clusters with the non-portable opt-in when the
    // device can hold one, else the portable 8
    RAS_CUDA(c, cudaFuncSetAttribute(k_trsv_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    c->trsv_cl_max = 8;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kNT_TRC);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k_trsv_cl, &cfg) == cudaSuccess && ncl > 0) c->trsv_cl_max = 16;
    cudaGetLastError();
    const char* f = getenv("RAS_TRSV_CL");
    const char* t = getenv("RAS_TRSV_CL_NT");
    c->trsv_cl_force = f ? std::max(1, std::min(c->trsv_cl_max, atoi(f))) : 0;
    c->trsv_cl_nt = t ? std::max(32, std::min(kNT_TRC, atoi(t))) : kNT_TRC;
    // DSMEM-routed solve where both factors qualify: one cluster size for every
    // launch (the routing depends on it): one row per thread where the widest level
    // allows, shrunk until all local subdomains' clusters are co-resident
    // (RAS_TRSV_DS_CL forces a size; RAS_TRSV=cl keeps k_trsv_cl)
    const char* fd = getenv("RAS_TRSV_DS_CL");
    const char* e = getenv("RAS_TRSV");
    c->trsv_cl_forced = (e && std::strcmp(e, "cl") == 0) || f;
    if (!(e && std::strcmp(e, "cl") == 0)) {
      RAS_CUDA(c, cudaFuncSetAttribute(k_trsv_ds, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      RAS_CUDA(c, cudaFuncSetAttribute(k_trsv_ds, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(2 * kTrdSlots * sizeof(double))));
      int32_t wide = 1;
      for (int32_t w : c->tri_f.sub_max_lev) wide = std::max(wide, w);
      for (int32_t w : c->tri_b.sub_max_lev) wide = std::max(wide, w);
      const int lo = (int)((wide + kTrdRows * kNT_TRD - 1) / (kTrdRows * kNT_TRD));
      const int want = std::min(c->trsv_cl_max, (int)((wide + kNT_TRD - 1) / kNT_TRD));
      int ncl = fd ? std::max(1, std::min(c->trsv_cl_max, atoi(fd))) : lo;
      if (!fd)
        for (int k = want; k >= lo; --k)
          if (trsv_ds_fit(c, k) >= c->nl) {
            ncl = k;
            break;
          }
      ras_status st = RAS_OK;
      if (lo <= c->trsv_cl_max && build_ds(c, F, ncl, c->tri_f, &st) && build_ds(c, B, ncl, c->tri_b, &st))
        c->trsv_ds = true;
      if (st != RAS_OK) return st;
      if (getenv("RAS_TRSV_DEBUG")) fprintf(stderr, "k_trsv_ds: %s, cluster %d\n", c->trsv_ds ? "on" : "off", ncl);
    }
  }
  if (c->trsv_sf) {  // arm y and z with the sentinel (the solves re-arm each other afterwards)
    k_trsv_arm<<<148 * 4, 256, 0, c->stream>>>(c->rows_pad, c->d_y, c->d_z);
    RAS_CUDA(c, cudaGetLastError());
    RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  c->ic = true;
  const double rows = (double)c->plan->rows_local;
  c->mb.update_dot = rows * (8 /*p*/ + 8 /*q*/ + 16 /*r*/ + 16 /*d*/);
  c->mb.pupdate = c->fuse_p ? 0.0 : rows * (8 /*z*/ + 16 /*p*/);
  c->mb.trsv = 0.5 * (c->tri_f.bytes + c->tri_b.bytes);
  c->mb.zdot = rows * 16.0;
  return RAS_OK;
}

// NEXT f1 setup: complete banded Cholesky factors on the host, uploaded once
static ras_status upload_band(ras_ctx* c) {
  const ras_plan* pl = c->plan;
  for (const auto& S : pl->subs)
    if (S.nrows_pad > kBandMaxRows)
      return set_err(c, RAS_EINVAL, "cholesky local solve: subdomain " + std::to_string(S.p) + " has " +
                                        std::to_string(S.nrows_pad) + " rows (max " + std::to_string(kBandMaxRows) + ")");
  int64_t total = 0;  // band entries, checked before factoring
  for (const auto& S : pl->subs) {
    int64_t b = 0;
    for (int64_t i = 0; i < S.nrows_pad; ++i)
      for (int64_t e = pl->Ap_ptr[S.row_off + i]; e < pl->Ap_ptr[S.row_off + i + 1]; ++e)
        b = std::max<int64_t>(b, std::llabs(i - (int64_t)pl->Ap_col[e]));
    total += S.nrows_pad * (b + 1);
  }
  if ((double)total * 16.0 > 16e9) return set_err(c, RAS_EINVAL, "cholesky local solve: bands exceed 16 GB");
  BandHost H;
  try {
    build_band_cholesky(pl, H);
  } catch (const Fail& f) {
    return set_err(c, f.st, f.msg);
  }
  double *L, *U, *binv;
  int64_t *off, *boff;
  int32_t* bw;
  // inverses of the 32 x 32 diagonal blocks of every L (forward substitution on
  // the host, FP64): the device applies them as dense products
  std::vector<int64_t> bo(pl->subs.size() + 1, 0);
  for (size_t lp = 0; lp < pl->subs.size(); ++lp) bo[lp + 1] = bo[lp] + pl->subs[lp].nrows_pad * 32;
  std::vector<double> bi((size_t)bo.back(), 0.0);
  for (size_t lp = 0; lp < pl->subs.size(); ++lp) {
    const int64_t n = pl->subs[lp].nrows_pad, b = H.bw[lp], wdt = b + 1;
    const double* Lb = H.L.data() + H.off[lp];
    for (int64_t k = 0; k < n / 32; ++k) {
      double T[32][32] = {}, X[32][32] = {};
      for (int l = 0; l < 32; ++l)
        for (int m = 0; m <= l; ++m) {
          const int64_t i = 32 * k + l, j = 32 * k + m;
          if (i - j <= b) T[l][m] = Lb[i * wdt + (j - i + b)];
        }
      for (int m = 0; m < 32; ++m) {  // column m of T^-1
        X[m][m] = 1.0 / T[m][m];
        for (int l = m + 1; l < 32; ++l) {
          double acc = 0.0;
          for (int t = m; t < l; ++t) acc += T[l][t] * X[t][m];
          X[l][m] = -acc / T[l][l];
        }
      }
      double* dst = bi.data() + bo[lp] + k * 1024;
      for (int l = 0; l < 32; ++l)
        for (int m = 0; m < 32; ++m) dst[l * 32 + m] = X[l][m];
    }
  }
  TRY(upload(c, &L, H.L, 1));
  TRY(upload(c, &U, H.U, 1));
  TRY(upload(c, &binv, bi, 1));
  TRY(upload(c, &boff, bo));
  TRY(upload(c, &off, H.off));
  TRY(upload(c, &bw, H.bw));
  c->band = BandDev{L, U, binv, boff, off, bw};
  int nmax = 0;
  for (const auto& S : pl->subs) nmax = std::max<int>(nmax, (int)S.nrows_pad);
  c->band_smem = (size_t)nmax * sizeof(double);
  TRY(allow_smem(c, (const void*)k_band_chol));
  c->chol = true;
  c->mb.band = 16.0 * (double)H.off.back() + (double)pl->rows_local * 12.0 + (double)pl->n_own * 16.0;
  return RAS_OK;
}

static ras_status upload_plan(ras_ctx* c) {
  ras_plan* pl = c->plan;
  c->rows_pad = pl->rows_pad;
  c->n_own = pl->n_own;
  c->n_halo = pl->n_halo;
  c->ntiles = (int64_t)pl->tile_sub.size();
  c->nl = (int32_t)pl->subs.size();
  TRY(upload(c, &c->d_b, pl->b_loc));
  TRY(upload(c, &c->d_own_slot, pl->own_slot));
  // Lane-packed SELL-Z (dictionary values, 16-bit column offsets) whenever the
  // matrix allows it, unless plain SELL is forced (options.matrix_format = 1);
  // the fused-p kernel reads the plain format.  Only one format lives on the
  // device.  Measured on B200 (round 1, C2): 7.9 ms/sweep SELL-Z vs 9.3 plain.
  c->z = pl->z_ok && !c->fuse_p && c->opt.matrix_format != 1;
  int64_t* sp;
  if (c->z) {
    double* tb;
    uint8_t *rc, *lc, *dc;
    int32_t *rk, *lk, *rw, *lw;
    uint16_t *rd, *ld;
    TRY(upload(c, &tb, pl->z_table, 1));
    TRY(upload(c, &dc, pl->D_code, 1));
    TRY(upload(c, &sp, pl->R_sptr));
    TRY(upload(c, &rc, pl->R_code, 1));
    TRY(upload(c, &rk, pl->R_kbase, 1));
    TRY(upload(c, &rd, pl->R_d16, 1));
    TRY(upload(c, &rw, pl->R_wide, 1));
    c->R = Sell{sp, nullptr, nullptr, rk, rd, rw, rc, tb};
    TRY(upload(c, &sp, pl->L_sptr));
    TRY(upload(c, &lc, pl->L_code, 1));
    TRY(upload(c, &lk, pl->L_kbase, 1));
    TRY(upload(c, &ld, pl->L_d16, 1));
    TRY(upload(c, &lw, pl->L_wide, 1));
    c->L = Sell{sp, nullptr, nullptr, lk, ld, lw, lc, tb};
    c->D = Diag{nullptr, dc, tb};
    c->zwR = pl->zR_w;
    c->zwL = pl->zL_w;
  } else {
    int32_t* ci;
    double* va;
    TRY(upload(c, &c->d_diag, pl->diag));
    TRY(upload(c, &sp, pl->R_sptr));
    TRY(upload(c, &ci, pl->R_col, 1));
    TRY(upload(c, &va, pl->R_val, 1));
    c->R = Sell{sp, ci, va, nullptr, nullptr, nullptr, nullptr, nullptr};
    TRY(upload(c, &sp, pl->L_sptr));
    TRY(upload(c, &ci, pl->L_col, 1));
    TRY(upload(c, &va, pl->L_val, 1));
    c->L = Sell{sp, ci, va, nullptr, nullptr, nullptr, nullptr, nullptr};
    c->D = Diag{c->d_diag, nullptr, nullptr};
  }
  c->wR = c->wL = 0;
  for (size_t s = 0; s + 1 < pl->R_sptr.size(); ++s) {
    c->wR = std::max<int>(c->wR, (int)((pl->R_sptr[s + 1] - pl->R_sptr[s]) / 32));
    c->wL = std::max<int>(c->wL, (int)((pl->L_sptr[s + 1] - pl->L_sptr[s]) / 32));
  }
  std::vector<int64_t> stb(c->nl);
  std::vector<int32_t> snt(c->nl);
  for (int i = 0; i < c->nl; ++i) {
    stb[i] = pl->subs[i].tile_begin;
    snt[i] = (int32_t)pl->subs[i].ntiles;
  }
  if (pl->tile_rows != kTileRows) return set_err(c, RAS_ESTATE, "plan tile_rows != kernel tile rows");
  std::vector<int4> tiles(pl->tile_sub.size());
  for (size_t i = 0; i < tiles.size(); ++i)
    tiles[i] = make_int4((int)pl->tile_row0[i], pl->tile_nrows[i], pl->tile_sub[i], 0);
  int4* ti;
  int64_t* sb;
  int32_t* sn;
  TRY(upload(c, &ti, tiles));
  TRY(upload(c, &sb, stb));
  TRY(upload(c, &sn, snt));
  c->T = Tiles{ti, sb, sn, c->ntiles};
  if (pl->stage_max != kStageMax) return set_err(c, RAS_ESTATE, "plan stage_max != kernel kStageMax");
  std::vector<int2> cspan(pl->tile_cmin.size());
  for (size_t i = 0; i < cspan.size(); ++i) cspan[i] = make_int2(pl->tile_cmin[i], pl->tile_clen[i]);
  TRY(upload(c, &c->d_cspan, cspan, 1));
  c->d_x = (double*)dalloc_raw(c, (size_t)(c->n_own + c->n_halo) * 8);
  if (!c->d_x) return set_err(c, RAS_ENOMEM, "device allocation failed (x storage)");
  TRY(zalloc(c, &c->d_r, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_p, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_p2, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_q, (size_t)c->rows_pad));
  TRY(zalloc(c, &c->d_d, (size_t)c->rows_pad));
  // Local-PCG execution path (ras_pcg_path): BLOCK when every local Omega_p fits
  // one CTA's shared memory (the paper's 4096-unknown regime, NEXT f2), else
  // RESIDENT when a cooperative grid can keep every subdomain on chip, else TILED.
  {
    int nmax = 0;
    std::vector<int32_t> ro(pl->subs.size()), nr(pl->subs.size());
    for (size_t i = 0; i < pl->subs.size(); ++i) {
      ro[i] = (int32_t)pl->subs[i].row_off;
      nr[i] = (int32_t)pl->subs[i].nrows_pad;
      nmax = std::max(nmax, nr[i]);
    }
    const int req = c->opt.pcg_path;
    if (req < RAS_PCG_AUTO || req > RAS_PCG_RESIDENT) return set_err(c, RAS_EINVAL, "unknown pcg_path");
    const bool jac = c->opt.local_solver == RAS_LS_JACOBI_PCG || c->opt.local_solver == RAS_LS_EXACT_PCG;
    const bool eligible = jac && !c->fuse_p && !c->stage;
    if (req != RAS_PCG_AUTO && req != RAS_PCG_TILED && !eligible)
      return set_err(c, RAS_EINVAL, "pcg_path BLOCK/RESIDENT need Jacobi or exact PCG without fuse_p/stage_p");
    c->small = eligible && nmax <= kSmallMaxRows && (req == RAS_PCG_AUTO || req == RAS_PCG_BLOCK);
    if (req == RAS_PCG_BLOCK && !c->small)
      return set_err(c, RAS_EINVAL, "pcg_path BLOCK needs every |Omega_p| <= 14336 rows (padded)");
    c->small_nmax = nmax;
    c->path = c->small ? RAS_PCG_BLOCK : RAS_PCG_TILED;
    int32_t *dro, *dnr;
    TRY(upload(c, &dro, ro));
    TRY(upload(c, &dnr, nr));
    c->SS = SmallSubs{dro, dnr};
    if (!c->small && eligible && (req == RAS_PCG_AUTO || req == RAS_PCG_RESIDENT)) TRY(setup_resident(c, nmax));
    if (req == RAS_PCG_RESIDENT && c->path != RAS_PCG_RESIDENT)
      return set_err(c, RAS_EINVAL, "pcg_path RESIDENT: a subdomain is too large for the cooperative grid");
  }
  const int nl = c->nl;
  TRY(zalloc(c, &c->S.rt2, nl));
  TRY(zalloc(c, &c->S.rho, nl));
  TRY(zalloc(c, &c->S.own2, nl));
  TRY(zalloc(c, &c->S.alpha, nl));
  TRY(zalloc(c, &c->S.beta, nl));
  TRY(zalloc(c, &c->S.rr, nl));
  TRY(zalloc(c, &c->S.active, nl));
  TRY(zalloc(c, &c->S.its, nl));
  TRY(zalloc(c, &c->S.ticket, nl));
  TRY(zalloc(c, &c->S.inner_total, nl));
  TRY(zalloc(c, &c->S.partials, (size_t)c->ntiles * kNP));
  TRY(zalloc(c, &c->d_stop, 1));
  TRY(zalloc(c, &c->d_sync, 1));
  TRY(zalloc(c, &c->d_r2_local, 1));
  TRY(zalloc(c, &c->d_r2_global, 1));
  TRY(zalloc(c, &c->d_nactive, 1));
  RAS_CUDA(c, cudaHostAlloc((void**)&c->h_stop, 32 * sizeof(int32_t), cudaHostAllocMapped));
  RAS_CUDA(c, cudaHostGetDevicePointer((void**)&c->h_stop_dev, c->h_stop, 0));
  RAS_CUDA(c, cudaHostAlloc((void**)&c->h_nactive, (size_t)(c->nl + 1) * 4, cudaHostAllocDefault));
  // exchange lists (sync): concatenated per peer
  c->send_off.assign(c->world + 1, 0);
  c->send_cnt.assign(c->world, 0);
  c->recv_off.assign(c->world, 0);
  c->recv_cnt.assign(c->world, 0);
  std::vector<int32_t> slots;
  for (int r = 0; r < c->world; ++r) {
    c->send_off[r] = (int64_t)slots.size();
    c->send_cnt[r] = (int64_t)pl->send_slot[r].size();
    slots.insert(slots.end(), pl->send_slot[r].begin(), pl->send_slot[r].end());
    c->recv_off[r] = pl->halo_off[r];
    c->recv_cnt[r] = pl->halo_off[r + 1] - pl->halo_off[r];
  }
  c->send_off[c->world] = (int64_t)slots.size();
  c->n_send = (int64_t)slots.size();
  TRY(upload(c, &c->d_send_slot, slots, 1));
  TRY(zalloc(c, &c->d_sendbuf, (size_t)std::max<int64_t>(c->n_send, 1)));
  compute_model_bytes(c);
  return RAS_OK;
}

static ras_status setup_impl(ras_ctx* c, const ras_csr* A, const double* b, const ras_partition* part, int32_t overlap,
                             const ras_comm* comm) {
  if (comm) {
    c->rank = comm->rank;
    c->world = comm->world;
    c->device = comm->device;
    c->dev_alloc = comm->dev_alloc;
    c->dev_free = comm->dev_free;
    c->alloc_user = comm->alloc_user;
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return set_err(c, RAS_EINVAL, "bad rank/world");
    if (c->world > 1 && !comm->nccl_unique_id)
      return set_err(c, RAS_EINVAL, "world > 1 needs nccl_unique_id (the loopback group key in loopback mode)");
    if (comm->transport != RAS_TRANSPORT_NCCL && comm->transport != RAS_TRANSPORT_LOOPBACK)
      return set_err(c, RAS_EINVAL, "unknown ras_comm.transport");
    c->loopback = c->world > 1 && comm->transport == RAS_TRANSPORT_LOOPBACK;
    RAS_CUDA(c, cudaSetDevice(c->device));
  } else {
    RAS_CUDA(c, cudaGetDevice(&c->device));
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_err(c, RAS_ESTATE, "no CUDA device visible");
  if (comm && comm->cuda_stream) {
    c->stream = (cudaStream_t)comm->cuda_stream;
  } else {
    RAS_CUDA(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  // ---- plan: overlap sets and index maps on the device (default) or the host ----
  const double ts0 = now_s();
  ras_status s = c->opt.device_setup ? plan_build_device(c, &c->plan, A, b, part, overlap)
                                     : ras_plan_build(&c->plan, A, b, part, overlap, c->rank, c->world);
  if (s != RAS_OK) return set_err(c, s, tls_error());
  c->setup_phase[0] = now_s() - ts0;
  if (c->world > 1) {
    if (c->loopback) {
      TRY(loop_join(c, comm->nccl_unique_id));
    } else {
      ncclUniqueId id;
      std::memcpy(&id, comm->nccl_unique_id, sizeof(id));
      RAS_NCCL(c, ncclCommInitRank(&c->nccl, c->world, id, c->rank));
    }
    TRY(exchange_requests(c));
  } else {
    // nothing to exchange: single rank
  }
  if (ras_plan_set_robin(c->plan, c->opt.robin) != RAS_OK)
    return set_err(c, RAS_EINVAL, "robin (ORAS transmission parameter) must be in [0, 1)");
  if (c->opt.robin > 0.0 && overlap < 1)
    return set_err(c, RAS_EINVAL, "robin > 0 (ORAS) needs overlap >= 1: without overlap the iteration diverges (R30)");
  const double ts1 = now_s();
  s = ras_plan_finalize(c->plan);
  if (s != RAS_OK) return set_err(c, s, tls_error());
  const double ts2 = now_s();
  TRY(upload_plan(c));
  c->setup_phase[1] = ts2 - ts1;
  c->setup_phase[2] = now_s() - ts2;
  // ||b||^2 over all ranks (owned rows), fixed order on one rank, NCCL sum across ranks
  c->b2_global = c->plan->b2_global_local;
  TRY(coll_allreduce_f64(c, &c->b2_global, 1, false));
  if (c->opt.local_solver == RAS_LS_IC0_PCG || c->opt.local_solver == RAS_LS_ILU0_PCG) {
    TRY(upload_factors(c));
  } else if (c->opt.local_solver == RAS_LS_CHOLESKY) {
    TRY(upload_band(c));
  } else if (c->opt.local_solver != RAS_LS_JACOBI_PCG && c->opt.local_solver != RAS_LS_EXACT_PCG) {
    return set_err(c, RAS_EINVAL, "unknown local solver");
  }
  const double ts3 = now_s();
  TRY(async_setup(c));
  RAS_CUDA(c, cudaDeviceSynchronize());
  c->setup_phase[3] = now_s() - ts3;
  if (getenv("RAS_SETUP_TRACE"))
    fprintf(stderr, "[ras setup rank %d] plan (overlap sets + maps, %s) %.3f s, finalize (matrices) %.3f s, "
                    "upload + kernel layouts %.3f s, async runtime %.3f s\n",
            c->rank, c->opt.device_setup ? "device" : "host", c->setup_phase[0], c->setup_phase[1], c->setup_phase[2],
            c->setup_phase[3]);
  return RAS_OK;
}

// ---------------------------------------------------------------------------
// Per-kernel CUDA-event timing (ras_kernel_timing): events recorded on the
// library stream around each launch; durations summed per kernel kind.
// ---------------------------------------------------------------------------
int kt_begin(ras_ctx* c, cudaStream_t s) {
  if (!c->kt.on || s != c->stream) return -1;
  KTimer& t = c->kt;
  while (t.used + 2 > t.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    t.pool.push_back(e);
  }
  const int idx = (int)t.used;
  t.used += 2;
  cudaEventRecord(t.pool[idx], s);
  return idx;
}

void kt_end(ras_ctx* c, cudaStream_t s, int kind, int idx) {
  ++c->launches;
  if (idx < 0) return;
  cudaEventRecord(c->kt.pool[idx + 1], s);
  c->kt.kind.push_back(kind);
}

static void kt_reset(ras_ctx* c) {
  c->kt.used = 0;
  c->kt.kind.clear();
  for (int k = 0; k < K_NKINDS; ++k) {
    c->kt.total_ms[k] = 0.0;
    c->kt.count[k] = 0;
  }
}

static void kt_collect(ras_ctx* c) {
  if (!c->kt.on) return;
  cudaStreamSynchronize(c->stream);
  for (size_t i = 0; i < c->kt.kind.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->kt.pool[2 * i], c->kt.pool[2 * i + 1]);
    c->kt.total_ms[c->kt.kind[i]] += ms;
    c->kt.count[c->kt.kind[i]] += 1;
  }
}

// every kernel launch goes through LAUNCH: counted, and event-timed when the
// timing mode is on and the launch is on the library stream (`s` in scope or c->stream)
#define LAUNCH_ON(strm, kind, ...)        \
  do {                                    \
    const int ti_ = kt_begin(c, (strm));  \
    __VA_ARGS__;                          \
    kt_end(c, (strm), (kind), ti_);       \
  } while (0)
#define LAUNCH(kind, ...) LAUNCH_ON(c->stream, kind, __VA_ARGS__)

// Programmatic dependent launch (sm_90+): the next kernel of the PCG chain is
// scheduled while the previous one drains; every kernel starts with
// griddepcontrol.launch_dependents + griddepcontrol.wait (kernels.cuh), so
// the data dependence is still the full completion of the predecessor.
static thread_local size_t g_launch_smem = 0;  // dynamic shared memory of the next KL launch
template <typename Kern, typename... Args>
static void pdl_launch(cudaStream_t s, unsigned grid, unsigned block, Kern k, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = g_launch_smem;
  g_launch_smem = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}
// clusters of k_trsv_cl of size k that fit the device at once (cached per k)
static int trsv_cl_fit(ras_ctx* c, int k) {
  if (c->trsv_cl_fit.empty()) c->trsv_cl_fit.assign(17, -1);
  if (c->trsv_cl_fit[k] < 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)k);
    cfg.blockDim = dim3(kNT_TRC);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)k;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_trsv_cl, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    c->trsv_cl_fit[k] = n;
    if (getenv("RAS_TRSV_DEBUG")) fprintf(stderr, "k_trsv_cl: %d co-resident clusters of %d CTAs\n", n, k);
  }
  return c->trsv_cl_fit[k];
}

// k_trsv_ds: cluster launch (+ PDL), receive slots in dynamic shared memory
static void ds_launch(cudaStream_t s, unsigned grid, unsigned ncl, TriDs T, int32_t lp_base, const double* in,
                      double* out, const int32_t* active, Ctl C) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kNT_TRD);
  cfg.dynamicSmemBytes = (size_t)2 * kTrdSlots * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = ncl;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, k_trsv_ds, T, lp_base, in, out, active, C);
}

// k_trsv_cl: cluster launch (+ PDL)
static void cl_launch(cudaStream_t s, unsigned grid, unsigned ncl, TriCl T, int32_t lp_base, int32_t ntu,
                      const double* in, double* out, const int32_t* active, Ctl C) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kNT_TRC);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = ncl;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, k_trsv_cl, T, lp_base, ntu, in, out, active, C);
}
#define KL(strm, kind, grid, block, KERNEL, ...) LAUNCH_ON(strm, kind, pdl_launch(strm, grid, block, KERNEL, __VA_ARGS__))

// ---------------------------------------------------------------------------
// Sync sweep (lock-step, P155-161, P376-387): stream-ordered on one stream.
// ---------------------------------------------------------------------------

static ras_status exchange(ras_ctx* c, Ctl C);

// ---------------------------------------------------------------------------
// Enqueue helpers shared by the sync sweep (all local subdomains batched on the
// library stream), the async loop (one subdomain on its own stream) and the
// scripted lock-step mode.  Range.lp < 0 = every local subdomain.
// ---------------------------------------------------------------------------
Range range_all(ras_ctx* c) { return Range{0, (unsigned)c->ntiles, -1}; }
Range range_sub(ras_ctx* c, int lp) {
  const auto& S = c->plan->subs[lp];
  return Range{S.tile_begin, (unsigned)S.ntiles, lp};
}

// a1+a2 (+ Jacobi PCG start)
// per-subdomain scalar step after a streaming kernel (one CTA per subdomain in R)
template <int OP>
static void enq_finish(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C, int m = 0, double inner_tol = 0.0) {
  const unsigned nsub = R.lp < 0 ? (unsigned)c->nl : (unsigned)R.nsub;
  KL(s, K_CTRL, nsub, kFinThreads, k_finish<OP>, R.lp < 0 ? 0 : R.lp, c->T, c->S, C, m, inner_tol);
}

// Streaming kernels walk the tiles alternately forwards and backwards, so each
// starts on the rows whose vectors the previous kernel left in L2.
static Tiles tiles_next(ras_ctx* c) {
  Tiles t = c->T;
  c->dir ^= 1;
#ifdef RAS_NOREV
  t.rev = 0;
#else
  t.rev = c->dir;
#endif
  return t;
}

// SELL width dispatch: the smallest unrolled width >= the matrix's widest slice
#define RAS_DISPATCH_W(w, CALL) \
  switch ((w) <= 4 ? 4 : (w) <= 5 ? 5 : (w) <= 6 ? 6 : (w) <= 7 ? 7 : (w) <= 8 ? 8 : 0) { \
    case 4: CALL(4); break;                                                                \
    case 5: CALL(5); break;                                                                \
    case 6: CALL(6); break;                                                                \
    case 7: CALL(7); break;                                                                \
    case 8: CALL(8); break;                                                                \
    default: CALL(0); break;                                                               \
  }

// SELL-Z packed widths are 4 or 8
#define RAS_DISPATCH_ZW(w, CALL) \
  if ((w) == 4) {                \
    CALL(4);                     \
  } else {                       \
    CALL(8);                     \
  }

ras_status enq_residual(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C) {
#define RAS_RES(JAC, W, Z)                                                                                  \
  KL(s, K_RES, R.ntiles, (Z) ? kNT_RES_Z : kNT_RES, (k_residual<JAC, W, Z>), R.tile_base, tiles_next(c), c->R, (const double*)c->d_b, \
     c->D, (const int32_t*)c->d_own_slot, (const double*)c->d_x, c->d_r, c->d_p, c->S, C)
#define RAS_RES_J0(W) RAS_RES(true, W, false)
#define RAS_RES_I0(W) RAS_RES(false, W, false)
#define RAS_RES_JZ(W) RAS_RES(true, W, true)
#define RAS_RES_IZ(W) RAS_RES(false, W, true)
  if (!c->ic) {
    if (c->z) {
      RAS_DISPATCH_ZW(c->zwR, RAS_RES_JZ);
    } else {
      RAS_DISPATCH_W(c->wR, RAS_RES_J0);
    }
    enq_finish<F_RES_JAC>(c, s, R, C);
  } else {
    if (c->z) {
      RAS_DISPATCH_ZW(c->zwR, RAS_RES_IZ);
    } else {
      RAS_DISPATCH_W(c->wR, RAS_RES_I0);
    }
    enq_finish<F_RES_IC>(c, s, R, C);
  }
#undef RAS_RES_IZ
#undef RAS_RES_JZ
#undef RAS_RES_I0
#undef RAS_RES_J0
#undef RAS_RES
  return RAS_OK;
}

// z = M^-1 in via the forward (L) and backward (L^T / U) level-scheduled solves
static ras_status enq_precond(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C, const double* in, double* z) {
  for (int dir = 0; dir < 2; ++dir) {
    const TriBuf& T = dir == 0 ? c->tri_f : c->tri_b;
    uint32_t* ctr = c->d_trsv_ctr + dir * (c->nl + 1) + (R.lp < 0 ? c->nl : R.lp);
    int32_t* done = T.d_lev_done;
    RAS_CUDA(c, cudaMemsetAsync(ctr, 0, 4, s));
    int32_t c0 = 0, nch = T.nchunks;
    if (R.lp >= 0) {
      c0 = T.sub_c0[R.lp];
      nch = T.sub_nc[R.lp];
    }
    if (c->trsv_sf) {
      // sync-free: forward in -> y (re-arms z), backward y -> z (re-arms y)
      const double* src = dir == 0 ? in : c->d_y;
      double* dst = dir == 0 ? c->d_y : z;
      double* rearm = dir == 0 ? z : c->d_y;
      static const int sf_grid = [] {  // A/B knob: CTAs of the sync-free solve (default 2 per SM)
        const char* e = getenv("RAS_TRSV_SF_CTAS");
        return e ? std::max(1, atoi(e)) : 148 * 2;
      }();
      const unsigned g = (unsigned)std::max(1, std::min(nch, sf_grid));
      KL(s, K_TRSV, g, kTrsvChunk, k_trsv_sf, T.dev, (int)(R.lp < 0), c0, nch, ctr, src, dst, rearm,
         (const int32_t*)c->S.active, C);
      continue;
    }
    if (c->trsv_ds) {
      // DSMEM-routed: one cluster of the routing's size per subdomain
      const int l0 = R.lp < 0 ? 0 : R.lp, nsub = R.lp < 0 ? c->nl : 1, ncl = T.ds_ncl;
      const double* src = dir == 0 ? in : c->d_q;
      double* dst = dir == 0 ? c->d_q : z;
      LAUNCH_ON(s, K_TRSV, ds_launch(s, (unsigned)(nsub * ncl), (unsigned)ncl, T.ds, (int32_t)l0, src, dst,
                                     (const int32_t*)c->S.active, C));
      continue;
    }
    if (c->trsv_cl_max > 0) {
      // cluster-resident: one cluster per subdomain, sized to the widest level
      const int l0 = R.lp < 0 ? 0 : R.lp, nsub = R.lp < 0 ? c->nl : 1;
      int32_t wide = 1;
      for (int lp = l0; lp < l0 + nsub; ++lp) wide = std::max(wide, T.sub_max_lev[lp]);
      // one row per thread where the widest level allows (up to kTrcRPT are
      // prefetched, more are fetched on the spot), shrunk until all nsub clusters
      // fit the GPU at once (no second wave of clusters)
      int ncl = c->trsv_cl_force;
      if (!ncl) {
        const int want = std::min(c->trsv_cl_max, (int)((wide + c->trsv_cl_nt - 1) / c->trsv_cl_nt));
        ncl = want;
        for (int k = want; k >= 1; --k)
          if (trsv_cl_fit(c, k) >= nsub) {
            ncl = k;
            break;
          }
      }
      // a level wider than kTrcRPT rows per thread of one cluster (one huge
      // subdomain, e.g. C4's 256^3 per GPU) would leave most SMs idle: the
      // grid-wide level-counter kernel below takes it (unless RAS_TRSV=cl)
      const bool too_wide = (int64_t)ncl * c->trsv_cl_nt * kTrcRPT < wide;
      if (!too_wide || c->trsv_cl_forced) {
      const double* src = dir == 0 ? in : c->d_q;
      double* dst = dir == 0 ? c->d_q : z;
      LAUNCH_ON(s, K_TRSV, cl_launch(s, (unsigned)(nsub * ncl), (unsigned)ncl, T.cl, (int32_t)l0, (int32_t)c->trsv_cl_nt, src, dst,
                                     (const int32_t*)c->S.active, C));
      continue;
      }
    }
    if (R.lp < 0) {
      RAS_CUDA(c, cudaMemsetAsync(done, 0, (size_t)T.nlev_slots * 4, s));
    } else {
      RAS_CUDA(c, cudaMemsetAsync(done + T.sub_lev_off[R.lp], 0, (size_t)T.sub_nlev[R.lp] * 4, s));
    }
    const unsigned g = (unsigned)std::max(1, std::min(nch, 148 * 8 * 256 / kTrsvChunk));
    const double* src = dir == 0 ? in : c->d_q;  // forward: in -> y (in q), backward: y -> z
    double* dst = dir == 0 ? c->d_q : z;
    if (T.cl_ok && c->trsv_mode != 1) {  // position-ordered operands prefetched across the level wait
      // the launch's chunk flags cleared in stream order (replay-safe inside the
      // async driver's captured graphs), completion = 1
      RAS_CUDA(c, cudaMemsetAsync(T.d_cflag + c0, 0, (size_t)nch * 4, s));
      KL(s, K_TRSV, g, kTrsvChunk, k_trsv_pf, T.dev, T.cl, (int)(R.lp < 0), c0, nch, ctr, (const int2*)T.d_cdep,
         T.d_cflag, 1, src, dst, (const int32_t*)c->S.active, C);
    } else {  // RAS_TRSV=level, or rows with > 4 dependencies
      KL(s, K_TRSV, g, kTrsvChunk, k_trsv, T.dev, (int)(R.lp < 0), c0, nch, ctr, done, src, dst,
         (const int32_t*)c->S.active, C);
    }
  }
  return RAS_OK;
}

static ras_status poll_inactive(ras_ctx* c, cudaStream_t s, const Range& R, bool* all_done) {
  if (R.lp < 0) {
    LAUNCH_ON(s, K_CTRL, k_count_active<<<1, 32, 0, s>>>(c->nl, c->S.active, c->d_nactive));
    RAS_CUDA(c, cudaMemcpyAsync(c->h_nactive + c->nl, c->d_nactive, 4, cudaMemcpyDeviceToHost, s));
    RAS_CUDA(c, cudaStreamSynchronize(s));
    *all_done = c->h_nactive[c->nl] == 0;
  } else {
    RAS_CUDA(c, cudaMemcpyAsync(c->h_nactive + R.lp, c->S.active + R.lp, 4, cudaMemcpyDeviceToHost, s));
    RAS_CUDA(c, cudaStreamSynchronize(s));
    *all_done = c->h_nactive[R.lp] == 0;
  }
  return RAS_OK;
}

// a3: local PCG solve (m iterations; exact mode polls every 16 iterations)
template <int RPT, int W, bool Z>
static void small_attr(ras_ctx* c) {
  static std::once_flag once;  // per instantiation; the cap (device maximum) is the same for every context
  std::call_once(once, [c] { allow_smem(c, (const void*)k_small_pcg<RPT, W, Z>); });
}

// f2 regime: one CTA runs a subdomain's whole PCG + prolongation (k_small_pcg)
static ras_status enq_small_pcg(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C, int m, double inner_tol) {
  const unsigned nsub = R.lp < 0 ? (unsigned)c->nl : 1u;
  const int lp0 = R.lp < 0 ? 0 : R.lp;
  const bool dl2 = c->small_nmax > kSmallSmemDRows;  // d in L2 (row space d_d) for the larger subdomains
  const size_t smem = (size_t)(dl2 ? 2 : 3) * c->small_nmax * sizeof(double);
  double* dglob = dl2 ? c->d_d : nullptr;
  const int rpt = (c->small_nmax + kNT_SMALL - 1) / kNT_SMALL;
#define RAS_SMALL(RPT, W, Z)                                                                                     \
  small_attr<RPT, W, Z>(c);                                                                                      \
  g_launch_smem = smem;                                                                                          \
  KL(s, K_SMALL, nsub, kNT_SMALL, (k_small_pcg<RPT, W, Z>), lp0, c->SS, c->L, c->D, (const double*)c->d_r,      \
     (const double*)c->d_p, (const int32_t*)c->d_own_slot, c->d_x, c->S, C, m, inner_tol, dglob)
#define RAS_SMALL_R(W, Z)              \
  if (rpt <= 2) {                      \
    RAS_SMALL(2, W, Z);                \
  } else if (rpt <= 4) {               \
    RAS_SMALL(4, W, Z);                \
  } else if (rpt <= 6) {               \
    RAS_SMALL(6, W, Z);                \
  } else if (rpt <= 9) {               \
    RAS_SMALL(9, W, Z);                \
  } else {                             \
    RAS_SMALL(14, W, Z);               \
  }
#define RAS_SMALL_Z(W) RAS_SMALL_R(W, true)
#define RAS_SMALL_0(W) RAS_SMALL_R(W, false)
  if (c->z) {
    RAS_DISPATCH_ZW(c->zwL, RAS_SMALL_Z);
  } else {
    RAS_DISPATCH_W(c->wL, RAS_SMALL_0);
  }
#undef RAS_SMALL_0
#undef RAS_SMALL_Z
#undef RAS_SMALL_R
#undef RAS_SMALL
  return RAS_OK;
}

// RESIDENT path: one cooperative launch runs every local subdomain's whole PCG
// + prolongation (k_resident_pcg), batched (sync) solves only.
static ras_status enq_resident_pcg(ras_ctx* c, cudaStream_t s, Ctl C, int32_t m, double inner_tol, int lp_first,
                                   int nsub_) {
  // every reduction slot starts empty (kSlotEmpty = all ones)
  RAS_CUDA(c, cudaMemsetAsync(c->d_resid_slots, 0xff,
                              (size_t)c->RC.ngroups * std::max(c->resid_lanes, 1) * 3 * kResidNV * c->RC.gs * 8, s));
  const bool v2 = c->resid_lanes > 0 && !(inner_tol > 0.0);
  const void* fn = v2 ? resident2_kernel(c->resid_rpt, c->zwL, c->resid_lanes, c->resid_pat)
                      : resident_kernel(c->resid_rpt, c->z, c->z ? c->zwL : c->wL, inner_tol > 0.0, c->resid_pat);
  int lp0 = lp_first, nsub = nsub_;
  const int32_t* own = c->d_own_slot;
  double* x = c->d_x;
  int32_t chunk_max = c->resid_chunk, glo = c->resid_glo, ghi = c->resid_ghi;
  int32_t ntable = c->z ? (int32_t)c->plan->z_table.size() : 0;
  void* args1[] = {&lp0, &nsub, &c->SS, &c->RC, &c->L,      &c->D,      &own, &x,  &c->S,
                   &C,   &m,    &inner_tol,     &chunk_max, &glo,       &ghi, &ntable};
  void* args2[] = {&lp0, &nsub, &c->SS, &c->RC, &c->L, &c->D, &own, &x, &c->S, &C, &m, &chunk_max, &glo, &ghi, &ntable};
  void** args = v2 ? args2 : args1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(c->RC.ngroups * c->RC.gs));
  cfg.blockDim = dim3(v2 ? kNT_R2 : kNT_RESID);
  cfg.dynamicSmemBytes = c->resid_smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int ti = kt_begin(c, s);
  RAS_CUDA(c, cudaLaunchKernelExC(&cfg, fn, args));
  kt_end(c, s, K_RESID, ti);
#ifdef RAS_RESID_TRACE
  if (const char* f = getenv("RAS_TRACE_FILE")) {
    static std::vector<unsigned long long> h(160 * 64 * 4);
    RAS_CUDA(c, cudaStreamSynchronize(s));
    RAS_CUDA(c, cudaMemcpyFromSymbol(h.data(), g_resid_trace, h.size() * 8));
    if (FILE* fp = fopen(f, "wb")) {
      fwrite(h.data(), 8, h.size(), fp);
      RAS_CUDA(c, cudaMemcpyFromSymbol(h.data(), g_red_trace, h.size() * 8));
      fwrite(h.data(), 8, h.size(), fp);
      fclose(fp);
    }
  }
#endif
  return RAS_OK;
}

ras_status enq_pcg(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C, int m, double inner_tol, bool exact) {
  const unsigned g = R.ntiles;
  const int64_t tb = R.tile_base;
  if (c->chol) {  // NEXT f1: direct solve, one CTA per subdomain (+ prolongation)
    g_launch_smem = c->band_smem;
    KL(s, K_BAND, R.lp < 0 ? (unsigned)c->nl : 1u, kNT_BAND, k_band_chol, R.lp < 0 ? 0 : R.lp, c->SS, c->band,
       (const double*)c->d_r, (const int32_t*)c->d_own_slot, c->d_x, c->S, C);
    return RAS_OK;
  }
  if (c->small) return enq_small_pcg(c, s, R, C, m, inner_tol);
  if (c->path == RAS_PCG_RESIDENT && (R.lp < 0 || c->resid_seq))
    return enq_resident_pcg(c, s, C, m, inner_tol, R.lp < 0 ? 0 : R.lp, R.lp < 0 ? c->nl : R.nsub);
  if (c->ic) {  // PCG start: z = M^-1 r, p = z, rho = r.z
    TRY(enq_precond(c, s, R, C, c->d_r, c->d_z));
    KL(s, K_ZDOT, g, kNT_STREAM, k_zdot<true>, tb, tiles_next(c), (const double*)c->d_r, (const double*)c->d_z, c->d_p, c->S, C);
    enq_finish<F_ZDOT0>(c, s, R, C);
  }
  for (int it = 1; it <= m; ++it) {
    const bool last = it == m;
    // p double buffer: iteration it writes p_new, reads p_old (p of it-1)
    double* p_new = c->fuse_p ? ((it & 1) ? c->d_p : c->d_p2) : c->d_p;
    const double* p_old = c->fuse_p ? ((it & 1) ? c->d_p2 : c->d_p) : c->d_p;
    const double* zr = c->ic ? c->d_z : c->d_r;
#define RAS_SPMV_V(W, IC, FIRST)                                                                                  \
  KL(s, K_SPMV, g, kThreads, (k_spmv_pdot<W, IC, FIRST>), tb, tiles_next(c), c->L, (const double*)c->d_diag, zr, p_old, \
     p_new, c->d_q, c->S, C)
#define RAS_SPMV_JF(W) RAS_SPMV_V(W, false, true)
#define RAS_SPMV_JN(W) RAS_SPMV_V(W, false, false)
#define RAS_SPMV_IF(W) RAS_SPMV_V(W, true, true)
#define RAS_SPMV_IN(W) RAS_SPMV_V(W, true, false)
#define RAS_SPMV_P(W, Z, STG)                                                                                     \
  KL(s, K_SPMV, g, kNT_SPMV, (k_spmv_dot<W, Z, STG>), tb, tiles_next(c), c->L, c->D, (const double*)p_new, c->d_q, \
     c->S, C, (const int2*)c->d_cspan)
#define RAS_SPMV_P0(W) RAS_SPMV_P(W, false, false)
#define RAS_SPMV_PZ(W) RAS_SPMV_P(W, true, false)
#define RAS_SPMV_S0(W) RAS_SPMV_P(W, false, true)
#define RAS_SPMV_SZ(W) RAS_SPMV_P(W, true, true)
    if (!c->fuse_p) {
      // p_new was written by the previous iteration's p update (or the PCG start)
      if (c->z) {
        if (c->stage) {
          RAS_DISPATCH_ZW(c->zwL, RAS_SPMV_SZ);
        } else {
          RAS_DISPATCH_ZW(c->zwL, RAS_SPMV_PZ);
        }
      } else {
        if (c->stage) {
          RAS_DISPATCH_W(c->wL, RAS_SPMV_S0);
        } else {
          RAS_DISPATCH_W(c->wL, RAS_SPMV_P0);
        }
      }
    } else if (!c->ic) {
      if (it == 1) {
        RAS_DISPATCH_W(c->wL, RAS_SPMV_JF);
      } else {
        RAS_DISPATCH_W(c->wL, RAS_SPMV_JN);
      }
    } else {
      if (it == 1) {
        RAS_DISPATCH_W(c->wL, RAS_SPMV_IF);
      } else {
        RAS_DISPATCH_W(c->wL, RAS_SPMV_IN);
      }
    }
#undef RAS_SPMV_SZ
#undef RAS_SPMV_S0
#undef RAS_SPMV_PZ
#undef RAS_SPMV_P0
#undef RAS_SPMV_P
#undef RAS_SPMV_IN
#undef RAS_SPMV_IF
#undef RAS_SPMV_JN
#undef RAS_SPMV_JF
#undef RAS_SPMV_V
    enq_finish<F_SPMV>(c, s, R, C);
    if (!c->ic) {
      if (c->z)
        KL(s, K_UPD, g, kNT_UPD, (k_update_dot<true, true>), tb, tiles_next(c), c->D, (const double*)p_new,
           (const double*)c->d_q, c->d_r, c->d_d, c->S, C);
      else
        KL(s, K_UPD, g, kNT_UPD, (k_update_dot<true, false>), tb, tiles_next(c), c->D, (const double*)p_new,
           (const double*)c->d_q, c->d_r, c->d_d, c->S, C);
      enq_finish<F_UPD_JAC>(c, s, R, C, m, inner_tol);
      if (!c->fuse_p && !last) {
        if (c->z)
          KL(s, K_PUPD, g, kNT_STREAM, k_pupdate<true>, tb, tiles_next(c), c->D, (const double*)c->d_r, c->d_p, c->S, C);
        else
          KL(s, K_PUPD, g, kNT_STREAM, k_pupdate<false>, tb, tiles_next(c), c->D, (const double*)c->d_r, c->d_p, c->S, C);
      }
    } else {
      KL(s, K_UPD, g, kNT_UPD, (k_update_dot<false, false>), tb, tiles_next(c), c->D, (const double*)p_new,
         (const double*)c->d_q, c->d_r, c->d_d, c->S, C);
      enq_finish<F_UPD_IC>(c, s, R, C, m, inner_tol);
      if (!last) {
        TRY(enq_precond(c, s, R, C, c->d_r, c->d_z));
        KL(s, K_ZDOT, g, kNT_STREAM, k_zdot<false>, tb, tiles_next(c), (const double*)c->d_r, (const double*)c->d_z, c->d_p, c->S, C);
        enq_finish<F_ZDOT>(c, s, R, C);
        if (!c->fuse_p) KL(s, K_PUPD, g, kNT_STREAM, k_pupdate_z, tb, tiles_next(c), (const double*)c->d_z, c->d_p, c->S, C);
      }
    }
    if (exact && it % 16 == 0) {
      bool done = false;
      TRY(poll_inactive(c, s, R, &done));
      if (done) break;
    }
  }
  return RAS_OK;
}

// a4
ras_status enq_prolong(ras_ctx* c, cudaStream_t s, const Range& R, Ctl C) {
  if (c->small || c->chol) return RAS_OK;  // k_small_pcg / k_band_chol prolong in the same kernel
  if (c->path == RAS_PCG_RESIDENT && (R.lp < 0 || c->resid_seq)) return RAS_OK;  // so does k_resident_pcg
  KL(s, K_PROL, R.ntiles, kNT_STREAM, k_prolong, R.tile_base, tiles_next(c), (const int32_t*)c->d_own_slot, (const double*)c->d_d,
     c->d_x, c->S, C);
  return RAS_OK;
}

// check_only: the sweep at k == max_iters only evaluates x^{max_iters} (the
// device stops there whatever the residual), so its local solve is not enqueued.
// Phase events of one sync sweep (ras_stats_t t_*): boundaries recorded on the
// library stream, read back when the host next waits on the sweep's slot.
struct PhaseEv {
  cudaEvent_t e[6];  // start | residual | convcheck | local solve | prolong | exchange
  int n = 0;         // boundaries recorded in the sweep (3 for a check-only sweep)
};

static void phase_collect(ras_ctx* c, PhaseEv& P) {
  double* t[5] = {&c->st.t_residual, &c->st.t_convcheck, &c->st.t_local_solve, &c->st.t_prolong, &c->st.t_exchange};
  for (int i = 0; i + 1 < P.n; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, P.e[i], P.e[i + 1]) == cudaSuccess) *t[i] += 1e-3 * ms;
  }
  P.n = 0;
}

static ras_status sync_sweep(ras_ctx* c, double tol, int64_t max_iters, int m, double inner_tol, bool exact, int slot,
                             bool check_only, PhaseEv& P) {
  Ctl C{c->d_stop, 0};
  const Range R = range_all(c);
  RAS_CUDA(c, cudaEventRecord(P.e[0], c->stream));
  // a1+a2
  TRY(enq_residual(c, c->stream, R, C));
  RAS_CUDA(c, cudaEventRecord(P.e[1], c->stream));
  // a6 (global criterion on x^k, P344-346)
  LAUNCH(K_CTRL, k_sum_own<<<1, 32, 0, c->stream>>>(c->nl, c->S.own2, c->d_r2_local));
  const double* r2g = c->d_r2_local;
  if (c->world > 1) {
    TRY(coll_allreduce(c, c->d_r2_local, c->d_r2_global, 1, ncclDouble, ncclSum, c->stream));
    r2g = c->d_r2_global;
  }
  LAUNCH(K_CTRL, k_sync_check<<<1, 32, 0, c->stream>>>(r2g, c->b2_global, tol, max_iters, c->d_sync, c->d_stop,
                                                       c->h_stop_dev + slot));
  RAS_CUDA(c, cudaEventRecord(P.e[2], c->stream));
  P.n = 3;
  if (check_only) return RAS_OK;
  // a3 (BLOCK / RESIDENT / direct: the prolongation is fused into the same launch)
  TRY(enq_pcg(c, c->stream, R, C, m, inner_tol, exact));
  RAS_CUDA(c, cudaEventRecord(P.e[3], c->stream));
  // a4
  TRY(enq_prolong(c, c->stream, R, C));
  RAS_CUDA(c, cudaEventRecord(P.e[4], c->stream));
  // a5
  TRY(exchange(c, C));
  RAS_CUDA(c, cudaEventRecord(P.e[5], c->stream));
  P.n = 6;
  RAS_CUDA(c, cudaGetLastError());
  return RAS_OK;
}

// a5 (sync, P376-387): pack + NCCL grouped send/recv straight into halo storage
// (no unpack: the receive buffer IS the halo segment of the peer's values).
static ras_status exchange(ras_ctx* c, Ctl C) {
  if (c->world == 1) return RAS_OK;
  if (c->n_send) {
    LAUNCH(K_PACK, k_pack<<<(unsigned)std::min<int64_t>((c->n_send + 255) / 256, 148 * 8), 256, 0, c->stream>>>(
                       c->n_send, c->d_send_slot, c->d_x, c->d_sendbuf, C));
  }
  std::vector<Xfer> snd, rcv;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (c->send_cnt[r]) snd.push_back(Xfer{r, c->d_sendbuf + c->send_off[r], (size_t)c->send_cnt[r]});
    if (c->recv_cnt[r]) rcv.push_back(Xfer{r, c->d_x + c->n_own + c->recv_off[r], (size_t)c->recv_cnt[r]});
  }
  return coll_sendrecv(c, snd, rcv, ncclFloat64, c->stream);
}

ras_status sync_exchange(ras_ctx* c) { return exchange(c, Ctl{nullptr, 0}); }

// True relative residual ||b - A x|| / ||b|| of the stored iterate (halo must be
// current): one residual pass over every tile + owned partial sums + allreduce.
ras_status global_residual(ras_ctx* c, double* rel) {
  Ctl C{nullptr, 0};
  TRY(enq_residual(c, c->stream, range_all(c), C));
  LAUNCH(K_CTRL, k_sum_own<<<1, 32, 0, c->stream>>>(c->nl, c->S.own2, c->d_r2_local));
  const double* r2g = c->d_r2_local;
  if (c->world > 1) {
    TRY(coll_allreduce(c, c->d_r2_local, c->d_r2_global, 1, ncclDouble, ncclSum, c->stream));
    r2g = c->d_r2_global;
  }
  double r2 = 0.0;
  RAS_CUDA(c, cudaMemcpyAsync(&r2, r2g, 8, cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  *rel = c->b2_global > 0.0 ? std::sqrt(r2) / std::sqrt(c->b2_global) : (r2 == 0.0 ? 0.0 : INFINITY);
  return RAS_OK;
}

static ras_status ensure_xglob(ras_ctx* c) {
  if (c->d_xglob) return RAS_OK;
  const ras_plan* pl = c->plan;
  std::vector<int32_t> og(pl->own_gid.begin(), pl->own_gid.end()), hg(pl->halo_gid.begin(), pl->halo_gid.end());
  TRY(upload(c, &c->d_own_gid, og, 1));
  TRY(upload(c, &c->d_halo_gid, hg, 1));
  c->d_xglob = (double*)dalloc(c, (size_t)pl->n * 8);
  if (!c->d_xglob) return set_err(c, RAS_ENOMEM, "device allocation failed (global x buffer)");
  if (c->world > 1) {
    // padded segment size and every rank's owned global ids, exchanged once
    double g = (double)c->n_own;
    TRY(coll_allreduce_f64(c, &g, 1, true));
    c->gmax = std::max<int64_t>((int64_t)g, 1);
    std::vector<int32_t> mine((size_t)c->gmax, -1);
    std::copy(og.begin(), og.end(), mine.begin());
    int32_t* d_mine;
    TRY(upload(c, &d_mine, mine));
    TRY(zalloc(c, &c->d_gid_all, (size_t)c->world * c->gmax));
    TRY(coll_allgather(c, d_mine, c->d_gid_all, (size_t)c->gmax, ncclInt32, c->stream));
    TRY(zalloc(c, &c->d_gsend, (size_t)c->gmax));
    TRY(zalloc(c, &c->d_grecv, (size_t)c->world * c->gmax));
  }
  return RAS_OK;
}

// x0 (host, global order) -> storage order on the device (one H2D copy + gather kernel)
static ras_status load_x0(ras_ctx* c, const double* x0) {
  const int64_t tot = c->n_own + c->n_halo;
  if (!x0) {
    RAS_CUDA(c, cudaMemsetAsync(c->d_x, 0, tot * 8, c->stream));
    return RAS_OK;
  }
  TRY(ensure_xglob(c));
  RAS_CUDA(c, cudaMemcpyAsync(c->d_xglob, x0, (size_t)c->plan->n * 8, cudaMemcpyHostToDevice, c->stream));
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 148 * 16));
  LAUNCH(K_CTRL, k_scatter_x0<<<g, 256, 0, c->stream>>>(c->n_own, c->n_halo, c->d_own_gid, c->d_halo_gid, c->d_xglob,
                                                         c->d_x));
  RAS_CUDA(c, cudaGetLastError());
  return RAS_OK;
}

// Gather owner values to x_out (len n) on every rank (P242).  One rank: owned
// storage -> global order on the device.  N ranks: one NCCL allgather of the
// owned values in padded per-rank segments (each rank receives only the other
// ranks' owned values, ~n words over NVLink), then one scatter into global order
// through the allgathered global ids (exchanged once); one D2H copy.
static ras_status gather(ras_ctx* c, double* x_out) {
  const ras_plan* pl = c->plan;
  TRY(ensure_xglob(c));
  if (c->world == 1) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((c->n_own + 255) / 256, 148 * 16));
    LAUNCH(K_CTRL, k_gather_x<<<g, 256, 0, c->stream>>>(c->n_own, c->d_own_gid, c->d_x, c->d_xglob));
  } else {
    RAS_CUDA(c, cudaMemcpyAsync(c->d_gsend, c->d_x, (size_t)c->n_own * 8, cudaMemcpyDeviceToDevice, c->stream));
    TRY(coll_allgather(c, c->d_gsend, c->d_grecv, (size_t)c->gmax, ncclFloat64, c->stream));
    const int64_t tot = (int64_t)c->world * c->gmax;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 148 * 16));
    LAUNCH(K_CTRL, k_gather_all<<<g, 256, 0, c->stream>>>(tot, c->d_gid_all, c->d_grecv, c->d_xglob));
  }
  RAS_CUDA(c, cudaMemcpyAsync(x_out, c->d_xglob, (size_t)pl->n * 8, cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  return RAS_OK;
}

static ras_status solve_sync(ras_ctx* c, double tol, int64_t max_iters) {
  const bool exact = c->opt.local_solver == RAS_LS_EXACT_PCG;
  int64_t max_rows = 0;
  for (auto& S : c->plan->subs) max_rows = std::max<int64_t>(max_rows, (int64_t)S.omega.size());
  const int m = exact ? (int)std::min<int64_t>(10 * max_rows, INT32_MAX / 2) : c->opt.inner_iters;
  const double inner_tol = exact ? 1e-14 : c->opt.inner_tol;
  // The host runs up to Q sweeps ahead of the device.  Before enqueuing sweep k
  // it waits for sweep k-Q and reads the stop flag AS OF sweep k-Q (ring slot
  // written by that sweep's check kernel), so every rank leaves the loop after
  // the same number of sweeps (matching NCCL calls) without a per-sweep sync.
  const int Q = std::max(1, c->opt.poll_interval);
  if (Q > 32) return set_err(c, RAS_EINVAL, "poll_interval must be <= 32");
  std::vector<cudaEvent_t> ev(Q);
  for (auto& e : ev) RAS_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  std::vector<PhaseEv> ph(Q);
  for (auto& P : ph)
    for (auto& e : P.e) RAS_CUDA(c, cudaEventCreate(&e));
  for (int i = 0; i < 32; ++i) c->h_stop[i] = 0;
  ras_status st = RAS_OK;
  for (int64_t k = 0;; ++k) {
    const int slot = (int)(k % Q);
    if (k >= Q) {
      if (cudaEventSynchronize(ev[slot]) != cudaSuccess) {
        st = cuda_err(c, cudaGetLastError(), "sweep");
        break;
      }
      phase_collect(c, ph[slot]);
      if (((volatile int32_t*)c->h_stop)[slot]) break;
    }
    if (k > max_iters) break;  // sweep max_iters only checks x^{max_iters}; the device stops there
    st = sync_sweep(c, tol, max_iters, m, inner_tol, exact, slot, k == max_iters, ph[slot]);
    if (st != RAS_OK) break;
    RAS_CUDA(c, cudaEventRecord(ev[slot], c->stream));
  }
  cudaStreamSynchronize(c->stream);
  for (auto& P : ph) {
    phase_collect(c, P);
    for (auto& e : P.e) cudaEventDestroy(e);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return st;
}

}  // namespace ras

using namespace ras;

extern "C" {

int32_t ras_abi_version(void) { return RAS_ABI_VERSION; }

#ifndef RAS_BUILD_HASH
#define RAS_BUILD_HASH "unstamped"
#endif
const char* ras_build_hash(void) { return RAS_BUILD_HASH; }

ras_status ras_options_default(ras_options* o) {
  if (!o) return RAS_EINVAL;
  std::memset(o, 0, sizeof(*o));
  o->local_solver = RAS_LS_JACOBI_PCG;
  o->inner_iters = 20;
  o->inner_tol = 0.0;
  o->detector = RAS_DET_DECENTRAL;
  o->max_resumes = 3;
  o->use_graphs = 1;
  o->poll_interval = 4;
  o->async_timeout_s = 1800.0;
  o->async_persistent = 2;
  o->device_setup = 1;
  return RAS_OK;
}

ras_status ras_setup(ras_ctx** out, const ras_csr* A, const double* b, const ras_partition* part, int32_t overlap,
                     const ras_options* opt, const ras_comm* comm) {
  if (!out) return set_err(nullptr, RAS_EINVAL, "ras_setup: out is NULL");
  *out = nullptr;
  const double t0 = now_s();
  ras_ctx* c = new ras_ctx();
  ras_options_default(&c->opt);
  if (opt) c->opt = *opt;
  if (c->opt.inner_iters < 1) c->opt.inner_iters = 1;
  c->fuse_p = c->opt.fuse_p != 0;
  c->stage = c->opt.stage_p != 0;
  if (c->opt.inner_tol < 0) {
    set_tls_error("inner_tol must be >= 0");
    delete c;
    return RAS_EINVAL;
  }
  ras_status s = setup_impl(c, A, b, part, overlap, comm);
  if (s != RAS_OK) {
    set_tls_error(c->err.empty() ? tls_error() : c->err);
    ras_free(c);
    return s;
  }
  c->setup_s = now_s() - t0;
  *out = c;
  return RAS_OK;
}

ras_status ras_set_rhs(ras_ctx* c, const double* b) {
  if (!c || !b) return RAS_EINVAL;
  RAS_CUDA(c, cudaSetDevice(c->device));
  ras_plan* pl = c->plan;
  std::vector<double> bl(pl->rows_pad, 0.0);
  // same accumulation order as the plan (per-subdomain sums, then the owned total)
  double b2 = 0.0;
  for (auto& S : pl->subs) {
    S.b2 = S.b2_owned = 0.0;
    for (int64_t i = 0; i < S.nrows; ++i) {
      const double v = b[S.omega[i] - pl->row_begin];
      bl[S.row_off + i] = v;
      S.b2 += v * v;
      if (S.owned[i]) S.b2_owned += v * v;
    }
    b2 += S.b2_owned;
  }
  pl->b_loc = bl;
  pl->b2_global_local = b2;
  RAS_CUDA(c, cudaMemcpyAsync(c->d_b, bl.data(), bl.size() * 8, cudaMemcpyHostToDevice, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  c->b2_global = b2;
  if (c->world > 1) TRY(coll_allreduce_f64(c, &c->b2_global, 1, false));
  // async Eq. 2 compares against the per-subdomain ||b~_p||^2 (or the owned-only variant)
  TRY(async_set_b2(c));
  return RAS_OK;
}

static ras_status solve_common(ras_ctx* c, double tol, int64_t max_iters, ras_mode mode) {
  if (!(tol > 0.0)) return set_err(c, RAS_EINVAL, "tol must be > 0");
  if (max_iters < 0) return set_err(c, RAS_EINVAL, "max_iters must be >= 0");
  RAS_CUDA(c, cudaSetDevice(c->device));
  std::memset(&c->st, 0, sizeof(c->st));
  SyncState z{};
  RAS_CUDA(c, cudaMemcpyAsync(c->d_sync, &z, sizeof(z), cudaMemcpyHostToDevice, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(c->d_stop, 0, 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(c->S.inner_total, 0, c->nl * 8, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(c->S.ticket, 0, c->nl * 4, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  ras_status s;
  if (mode == RAS_SYNC) {
    s = solve_sync(c, tol, max_iters);
    if (s != RAS_OK) return s;
    SyncState h{};
    RAS_CUDA(c, cudaMemcpy(&h, c->d_sync, sizeof(h), cudaMemcpyDeviceToHost));
    c->st.converged = h.converged;
    c->st.verified = h.converged;
    c->st.sweeps = h.sweeps;
    c->st.final_rel_residual = h.rel;
    c->updates.assign(c->nl, h.sweeps);
    c->st.updates_min = c->st.updates_median = c->st.updates_max = h.sweeps;
  } else if (mode == RAS_ASYNC) {
    s = solve_async(c, tol, max_iters);
    if (s != RAS_OK && s != RAS_ENOCONV && s != RAS_EVERIFY) return s;
    if (s != RAS_OK) return s;
  } else {
    return set_err(c, RAS_EINVAL, "unknown mode");
  }
  return RAS_OK;
}

static void finish_stats(ras_ctx* c, ras_mode mode, double t) {
  c->st.mode = mode;
  if (mode == RAS_SYNC) c->st.time_to_solution_s = t;  // async sets it at observed stop (R26)
  c->st.setup_s = c->setup_s;
  c->st.num_subdomains = c->plan->P;
  c->st.world = c->world;
  c->st.local_subdomains = c->nl;
  // the path both modes ran on: async BLOCK-sized subdomains use k_small_pcg (streams)
  // or its block_pcg (persistent kernel), RESIDENT-sized ones the sequential on-chip
  // schedule (R34), everything else the streaming kernels
  c->st.pcg_path = c->chol ? RAS_PCG_BLOCK : c->ic ? RAS_PCG_TILED : c->path;
  c->st.resident_pattern = c->path == RAS_PCG_RESIDENT && c->resid_pat;
  c->st.resident_lanes = c->path == RAS_PCG_RESIDENT ? c->resid_lanes : 0;
  c->st.rows_local = c->plan->rows_local;
  c->st.halo_values = c->n_halo;
  c->st.kernel_launches = c->launches;
  std::vector<int64_t> it(c->nl, 0);
  cudaMemcpy(it.data(), c->S.inner_total, c->nl * 8, cudaMemcpyDeviceToHost);
  c->st.inner_iters_total = std::accumulate(it.begin(), it.end(), (int64_t)0);
  // algorithmic bytes: per sweep residual + prolong + pack; per
  // PCG iteration of subdomain p the three passes over its |Omega_p| rows
  double frac_iters = 0.0;
  const double rows = (double)std::max<int64_t>(c->plan->rows_local, 1);
  for (int i = 0; i < c->nl; ++i) frac_iters += (double)it[i] * (double)c->plan->subs[i].nrows / rows;
  c->st.model_bytes = (double)c->st.sweeps * (c->mb.residual + c->mb.prolong + c->mb.pack + (c->chol ? c->mb.band : 0.0)) +
                      frac_iters * (c->mb.spmv_dot + c->mb.update_dot + c->mb.pupdate +
                                    (c->ic ? 2.0 * c->mb.trsv + c->mb.zdot : 0.0));
}

ras_status ras_solve(ras_ctx* c, double tol, int64_t max_iters, ras_mode mode, const double* x0, double* x_out) {
  if (!c) return set_err(nullptr, RAS_EINVAL, "ras_solve: ctx is NULL");
  const double t0 = now_s();
  RAS_CUDA(c, cudaSetDevice(c->device));
  c->launches = 0;
  kt_reset(c);
  TRY(load_x0(c, x0));
  ras_status s = solve_common(c, tol, max_iters, mode);
  if (s != RAS_OK && s != RAS_ENOCONV && s != RAS_EVERIFY) return s;
  const double t1 = now_s();
  if (x_out) TRY(gather(c, x_out));
  finish_stats(c, mode, t1 - t0);
  kt_collect(c);
  if (s != RAS_OK) return s;
  return c->st.converged ? RAS_OK : RAS_ENOCONV;
}

ras_status ras_solve_device(ras_ctx* c, double tol, int64_t max_iters, ras_mode mode, const double* x0_owned_dev,
                            double* x_owned_dev) {
  if (!c) return set_err(nullptr, RAS_EINVAL, "ras_solve_device: ctx is NULL");
  RAS_CUDA(c, cudaSetDevice(c->device));
  const double t0 = now_s();
  c->launches = 0;
  kt_reset(c);
  if (x0_owned_dev) {
    RAS_CUDA(c, cudaMemcpyAsync(c->d_x, x0_owned_dev, c->n_own * 8, cudaMemcpyDefault, c->stream));
  } else {
    RAS_CUDA(c, cudaMemsetAsync(c->d_x, 0, c->n_own * 8, c->stream));
  }
  if (c->n_halo) {
    if (x0_owned_dev && c->world > 1) {
      TRY(sync_exchange(c));  // halo = neighbours' owned x0 values
    } else {
      RAS_CUDA(c, cudaMemsetAsync(c->d_x + c->n_own, 0, c->n_halo * 8, c->stream));
    }
  }
  ras_status s = solve_common(c, tol, max_iters, mode);
  if (s != RAS_OK && s != RAS_ENOCONV && s != RAS_EVERIFY) return s;
  finish_stats(c, mode, now_s() - t0);
  if (x_owned_dev) RAS_CUDA(c, cudaMemcpyAsync(x_owned_dev, c->d_x, c->n_own * 8, cudaMemcpyDefault, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  kt_collect(c);
  if (s != RAS_OK) return s;
  return c->st.converged ? RAS_OK : RAS_ENOCONV;
}

int64_t ras_owned_count(const ras_ctx* c) { return c ? c->n_own : -1; }

ras_status ras_kernel_timing(ras_ctx* c, int32_t enable) {
  if (!c) return RAS_EINVAL;
  c->kt.on = enable != 0;
  return RAS_OK;
}

ras_status ras_kernel_times(const ras_ctx* c, ras_kernel_time_t* out, int32_t max_entries, int32_t* n_out) {
  if (!c || !n_out) return RAS_EINVAL;
  const char* names[K_NKINDS] = {"k_residual", "k_spmv_dot", c->ic ? "k_update_dot<ic>" : "k_update_dot",
                                 c->ic ? "k_pupdate_z" : "k_pupdate", "k_prolong", "k_pack", "control",
                                 "k_trsv", "k_zdot", "k_small_pcg", c->resid_lanes ? "k_resident2" : "k_resident_pcg",
                                 "k_band_chol"};
  const double bytes[K_NKINDS] = {c->mb.residual, c->mb.spmv_dot, c->mb.update_dot, c->mb.pupdate,
                                  c->mb.prolong,  c->mb.pack,     0.0,              c->mb.trsv,
                                  c->mb.zdot,     c->mb.local_solve, c->mb.local_solve, c->mb.band};
  int n = 0;
  for (int k = 0; k < K_NKINDS && n < max_entries; ++k) {
    if (!out) break;
    std::memset(&out[n], 0, sizeof(out[n]));
    std::strncpy(out[n].name, names[k], sizeof(out[n].name) - 1);
    out[n].launches = c->kt.count[k];
    out[n].total_ms = c->kt.total_ms[k];
    out[n].bytes_per_launch = bytes[k];
    ++n;
  }
  *n_out = out ? n : K_NKINDS;
  return RAS_OK;
}

ras_status ras_owned_gids(const ras_ctx* c, int64_t* g) {
  if (!c || !g) return RAS_EINVAL;
  std::copy(c->plan->own_gid.begin(), c->plan->own_gid.end(), g);
  return RAS_OK;
}

ras_status ras_stats(const ras_ctx* c, ras_stats_t* out) {
  if (!c || !out) return RAS_EINVAL;
  *out = c->st;
  return RAS_OK;
}

ras_status ras_update_counts(const ras_ctx* c, int64_t* out) {
  if (!c || !out) return RAS_EINVAL;
  for (int i = 0; i < c->nl; ++i) out[i] = i < (int)c->updates.size() ? c->updates[i] : 0;
  return RAS_OK;
}

void ras_free(ras_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  async_free(c);
  for (auto e : c->kt.pool) cudaEventDestroy(e);
  for (auto& b : c->bufs) {
    if (c->dev_free && !b.raw)
      c->dev_free(b.ptr, c->alloc_user);
    else
      cudaFree(b.ptr);
  }
  if (c->h_stop) cudaFreeHost(c->h_stop);
  if (c->h_nactive) cudaFreeHost(c->h_nactive);
  if (c->nccl) ncclCommDestroy(c->nccl);
  loop_leave(c);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  ras_plan_free(c->plan);
  delete c;
}

const char* ras_last_error(const ras_ctx* c) {
  if (!c) return tls_error().c_str();
  return c->err.c_str();
}

ras_status ras_nccl_unique_id(void* out128) {
  if (!out128) return RAS_EINVAL;
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    set_tls_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    return RAS_ENCCL;
  }
  std::memcpy(out128, &id, sizeof(id));
  return RAS_OK;
}

ras_status ras_ctx_plan(const ras_ctx* c, const ras_plan** out) {
  if (!c || !out) return RAS_EINVAL;
  *out = c->plan;
  return RAS_OK;
}

ras_status ras_set_scripted_flags(ras_ctx* c, const uint8_t* flags, int64_t nsweeps) {
  if (!c || (!flags && nsweeps)) return RAS_EINVAL;
  c->scripted.assign(flags, flags + nsweeps * c->nl);
  c->scripted_sweeps = nsweeps;
  return RAS_OK;
}

ras_status ras_debug_put_stress(ras_ctx* c, int64_t epochs, int64_t words, int64_t* out4) {
  if (!c || !out4) return RAS_EINVAL;
  RAS_CUDA(c, cudaSetDevice(c->device));
  return put_stress(c, epochs, words, out4);
}

ras_status ras_detector_stops(const ras_ctx* c, int64_t* out) {
  if (!c || !out) return RAS_EINVAL;
  for (int i = 0; i < c->nl; ++i) out[i] = i < (int)c->det_stops.size() ? c->det_stops[i] : -1;
  return RAS_OK;
}

}  // extern "C"
