// Incomplete factorizations of the local matrices A_p and their level sets
// (scope row a3', setup part).  Pure host C++, run once in ras_setup.
//
// PAPER §3.3.1 (P311-323): the local solve factors the local matrix once and
// solves triangular systems every iteration with a level-set strategy
// (cuSPARSE csrsm2).  Here the factors are the incomplete ones of the
// north_star: IC(0) in natural Omega_p order on the pattern of lower(A_p) (R9)
// and ILU(0) on the pattern of A_p (IKJ, R10).  Rows are grouped into levels
// (level = 1 + max level of the rows it depends on) and cut into 256-row
// chunks; the device solve processes chunks in level order (trsv.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "plan_internal.h"

namespace ras {

#ifndef RAS_TRSV_CHUNK
#define RAS_TRSV_CHUNK 256  // rows per level chunk = threads per CTA of the chunked trisolves (kernels.cuh)
#endif
static constexpr int kChunk = RAS_TRSV_CHUNK;

namespace {

struct RowList {  // sparse rows, columns ascending (subdomain-relative)
  std::vector<int64_t> ptr{0};
  std::vector<int32_t> col;
  std::vector<double> val;
  void push(const std::vector<std::pair<int32_t, double>>& r) {
    for (auto& e : r) {
      col.push_back(e.first);
      val.push_back(e.second);
    }
    ptr.push_back((int64_t)col.size());
  }
};

// IC(0): L (strict lower) rows + diagonal.  Sums in ascending k (as the oracle).
void ic0(const ras_plan* pl, int64_t r0, int64_t n, int32_t p, RowList& Ls, std::vector<double>& d) {
  d.assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = pl->Ap_ptr[r0 + i], b = pl->Ap_ptr[r0 + i + 1];
    std::vector<std::pair<int32_t, double>> Li;
    double aii = 0.0;
    for (int64_t e = a; e < b; ++e) {
      const int32_t j = pl->Ap_col[e];
      const double v = pl->Ap_val[e];
      if (j < i) {
        double s = v;
        // sum_{k<j, (i,k),(j,k) in P} L_ik L_jk : merge Li (all k < j) with row j
        size_t x = 0;
        int64_t y = Ls.ptr[j];
        const int64_t ye = Ls.ptr[j + 1];
        double acc = 0.0;
        while (x < Li.size() && y < ye) {
          if (Li[x].first == Ls.col[y]) {
            acc += Li[x].second * Ls.val[y];
            ++x;
            ++y;
          } else if (Li[x].first < Ls.col[y]) {
            ++x;
          } else {
            ++y;
          }
        }
        s -= acc;
        Li.emplace_back(j, s / d[j]);
      } else if (j == i) {
        aii = v;
      }
    }
    double sq = 0.0;
    for (auto& e : Li) sq += e.second * e.second;
    const double piv = aii - sq;
    if (!(piv > 0.0))
      throw Fail{RAS_ENOTSPD, "subdomain " + std::to_string(p) + ": IC(0) pivot " + std::to_string(piv) +
                                  " <= 0 at local row " + std::to_string(i)};
    d[i] = std::sqrt(piv);
    Ls.push(Li);
  }
}

// ILU(0), IKJ variant: L unit lower (strict part stored), U upper (strict + diag).
void ilu0(const ras_plan* pl, int64_t r0, int64_t n, int32_t p, RowList& Ls, RowList& Us, std::vector<double>& du) {
  du.assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = pl->Ap_ptr[r0 + i], b = pl->Ap_ptr[r0 + i + 1];
    std::vector<int32_t> cols(pl->Ap_col.begin() + a, pl->Ap_col.begin() + b);
    std::vector<double> w(pl->Ap_val.begin() + a, pl->Ap_val.begin() + b);
    auto find = [&](int32_t c) -> int {
      for (size_t t = 0; t < cols.size(); ++t)
        if (cols[t] == c) return (int)t;
      return -1;
    };
    for (size_t t = 0; t < cols.size() && cols[t] < i; ++t) {
      const int32_t k = cols[t];
      w[t] = w[t] / du[k];
      for (int64_t e = Us.ptr[k]; e < Us.ptr[k + 1]; ++e) {
        const int f = find(Us.col[e]);
        if (f >= 0) w[f] -= w[t] * Us.val[e];
      }
    }
    std::vector<std::pair<int32_t, double>> Lr, Ur;
    for (size_t t = 0; t < cols.size(); ++t) {
      if (cols[t] < i)
        Lr.emplace_back(cols[t], w[t]);
      else if (cols[t] == i)
        du[i] = w[t];
      else
        Ur.emplace_back(cols[t], w[t]);
    }
    if (!(du[i] > 0.0))
      throw Fail{RAS_ENOTSPD, "subdomain " + std::to_string(p) + ": ILU(0) pivot " + std::to_string(du[i]) +
                                  " <= 0 at local row " + std::to_string(i)};
    Ls.push(Lr);
    Us.push(Ur);
  }
}

}  // namespace

// Level-ordered triangular factor of every local subdomain (see plan_internal.h).
static void add_tri(const ras_plan* pl, int lp, const RowList& M, const std::vector<double>& diag, bool lower,
                    TriHost& T) {
  const auto& S = pl->subs[lp];
  const int64_t n = S.nrows_pad;
  std::vector<int32_t> lev(n, 0);
  int32_t nlev = 1;
  if (lower) {
    for (int64_t i = 0; i < n; ++i) {
      int32_t l = 0;
      for (int64_t e = M.ptr[i]; e < M.ptr[i + 1]; ++e) l = std::max(l, lev[M.col[e]] + 1);
      lev[i] = l;
      nlev = std::max(nlev, l + 1);
    }
  } else {
    for (int64_t i = n - 1; i >= 0; --i) {
      int32_t l = 0;
      for (int64_t e = M.ptr[i]; e < M.ptr[i + 1]; ++e) l = std::max(l, lev[M.col[e]] + 1);
      lev[i] = l;
      nlev = std::max(nlev, l + 1);
    }
  }
  // counting sort by level (rows ascending within a level)
  std::vector<int64_t> cnt(nlev + 1, 0);
  for (int64_t i = 0; i < n; ++i) cnt[lev[i] + 1]++;
  for (int32_t l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1), order(n);
  for (int64_t i = 0; i < n; ++i) order[pos[lev[i]]++] = i;
  const int64_t base = (int64_t)T.rows.size();
  T.sub_lev_off.push_back((int32_t)T.lev_nchunks.size());
  T.sub_nlev.push_back(nlev);
  T.sub_chunk_begin.push_back((int32_t)T.chunk.size());
  T.sub_pos_off.push_back((int32_t)T.lev_pos.size());
  int64_t maxlev = 0;
  for (int32_t l = 0; l <= nlev; ++l) T.lev_pos.push_back((int32_t)(base + cnt[l]));
  for (int32_t l = 0; l < nlev; ++l) maxlev = std::max<int64_t>(maxlev, cnt[l + 1] - cnt[l]);
  T.sub_max_lev.push_back((int32_t)maxlev);
  for (int64_t i = 0; i < n; ++i) T.max_deps = std::max<int32_t>(T.max_deps, (int32_t)(M.ptr[i + 1] - M.ptr[i]));
  for (int32_t l = 0; l < nlev; ++l) {
    int32_t nch = 0;
    for (int64_t a = cnt[l]; a < cnt[l + 1]; a += kChunk) {
      const int64_t b = std::min<int64_t>(a + kChunk, cnt[l + 1]);
      T.chunk.push_back({(int32_t)(base + a), (int32_t)(base + b), lp, l});
      ++nch;
    }
    T.lev_nchunks.push_back(nch);
  }
  T.sub_chunk_end.push_back((int32_t)T.chunk.size());
  T.max_levels = std::max<int64_t>(T.max_levels, nlev);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = order[k];
    T.rows.push_back((int32_t)(S.row_off + i));
    for (int64_t e = M.ptr[i]; e < M.ptr[i + 1]; ++e) {
      T.col.push_back((int32_t)(S.row_off + M.col[e]));
      T.val.push_back(M.val[e]);
    }
    T.rp.push_back((int32_t)T.col.size());
    T.diag[S.row_off + i] = diag[i];
  }
}

void build_factors(ras_plan* pl, int kind, TriHost& F, TriHost& B) {
  F = TriHost();
  B = TriHost();
  F.diag.assign(pl->rows_pad, 1.0);
  B.diag.assign(pl->rows_pad, 1.0);
  for (int lp = 0; lp < (int)pl->subs.size(); ++lp) {
    const auto& S = pl->subs[lp];
    const int64_t n = S.nrows_pad;
    RowList Ls, Us;
    std::vector<double> dL, dU;
    if (kind == RAS_LS_IC0_PCG) {
      ic0(pl, S.row_off, n, S.p, Ls, dL);
      // U = L^T (strict part) by transposition, diag the same
      std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t e = Ls.ptr[i]; e < Ls.ptr[i + 1]; ++e) rows[Ls.col[e]].emplace_back((int32_t)i, Ls.val[e]);
      for (auto& r : rows) Us.push(r);  // columns ascending: i visited ascending
      dU = dL;
    } else {
      ilu0(pl, S.row_off, n, S.p, Ls, Us, dU);
      dL.assign(n, 1.0);
    }
    add_tri(pl, lp, Ls, dL, true, F);
    add_tri(pl, lp, Us, dU, false, B);
  }
  // batched order: chunks sorted by (level, subdomain, position)
  for (TriHost* T : {&F, &B}) {
    T->batched.resize(T->chunk.size());
    for (size_t i = 0; i < T->chunk.size(); ++i) T->batched[i] = (int32_t)i;
    std::stable_sort(T->batched.begin(), T->batched.end(), [&](int32_t a, int32_t b) {
      const auto &x = T->chunk[a], &y = T->chunk[b];
      return x[3] != y[3] ? x[3] < y[3] : (x[2] != y[2] ? x[2] < y[2] : x[0] < y[0]);
    });
    T->rp.insert(T->rp.begin(), 0);
  }
}



// ---------------------------------------------------------------------------
// NEXT f1: complete (direct) Cholesky factor of every local A_p, banded.
// PAPER §3.3.1 (P311-318): the local matrix is factored once (CHOLMOD) and every
// local solve is two triangular solves.  A_p in natural Omega_p order is banded
// (2D tile: bandwidth ~ tile width + 2 gamma), so its complete factor L has all
// fill inside the band: L = chol(A_p) row by row (Crout / up-looking),
//   L(i,j) = (A(i,j) - sum_{k<j} L(i,k) L(j,k)) / L(j,j),  j in [i-b, i)
//   L(i,i) = sqrt(A(i,i) - sum_{k<i} L(i,k)^2)
// with sums in ascending k.  Stored twice, row-major with b+1 slots per row so
// both device solves read rows contiguously: lower band L (slot j - i + b) for
// the forward solve, upper band U = L^T (slot j - i) for the backward solve.
// Padding rows of the row space are identity rows.  Throws Fail on a pivot <= 0.
// ---------------------------------------------------------------------------
void build_band_cholesky(const ras_plan* pl, BandHost& H) {
  const size_t nl = pl->subs.size();
  H.off.assign(nl + 1, 0);
  H.bw.assign(nl, 0);
  for (size_t lp = 0; lp < nl; ++lp) {
    const auto& S = pl->subs[lp];
    int32_t b = 0;
    for (int64_t i = 0; i < S.nrows_pad; ++i)
      for (int64_t e = pl->Ap_ptr[S.row_off + i]; e < pl->Ap_ptr[S.row_off + i + 1]; ++e)
        b = std::max<int32_t>(b, (int32_t)std::llabs(i - (int64_t)pl->Ap_col[e]));
    H.bw[lp] = b;
    H.off[lp + 1] = H.off[lp] + S.nrows_pad * (int64_t)(b + 1);
  }
  H.L.assign((size_t)H.off[nl], 0.0);
  H.U.assign((size_t)H.off[nl], 0.0);
  std::vector<std::string> err(nl);
  auto factor = [&](size_t lp) {
    const auto& S = pl->subs[lp];
    const int64_t n = S.nrows_pad, b = H.bw[lp], w = b + 1;
    double* L = H.L.data() + H.off[lp];
    // band of A (lower part) into L, then factor in place
    for (int64_t i = 0; i < n; ++i)
      for (int64_t e = pl->Ap_ptr[S.row_off + i]; e < pl->Ap_ptr[S.row_off + i + 1]; ++e) {
        const int64_t j = pl->Ap_col[e];
        if (j <= i) L[i * w + (j - i + b)] = pl->Ap_val[e];
      }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t j0 = std::max<int64_t>(0, i - b);
      for (int64_t j = j0; j < i; ++j) {
        double s = L[i * w + (j - i + b)];
        for (int64_t k = std::max(j0, j - b); k < j; ++k) s -= L[i * w + (k - i + b)] * L[j * w + (k - j + b)];
        L[i * w + (j - i + b)] = s / L[j * w + b];
      }
      double s = L[i * w + b];
      for (int64_t k = j0; k < i; ++k) s -= L[i * w + (k - i + b)] * L[i * w + (k - i + b)];
      if (!(s > 0.0)) {
        err[lp] = "subdomain " + std::to_string(S.p) + ": Cholesky pivot " + std::to_string(s) + " <= 0 (local row " +
                  std::to_string(i) + ")";
        return;
      }
      L[i * w + b] = std::sqrt(s);
    }
    double* U = H.U.data() + H.off[lp];
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = std::max<int64_t>(0, i - b); j <= i; ++j) U[j * w + (i - j)] = L[i * w + (j - i + b)];
  };
  const size_t nt = std::max<size_t>(1, std::min<size_t>(nl, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t lp = t; lp < nl; lp += nt) factor(lp);
    });
  for (auto& t : th) t.join();
  for (size_t lp = 0; lp < nl; ++lp)
    if (!err[lp].empty()) throw Fail{RAS_ENOTSPD, err[lp]};
}

}  // namespace ras
