// Host-side setup plan (scope row a0): partition bookkeeping, gamma-hop overlap,
// ghosts, storage / restrict / prolong / pack maps, SELL-32 matrices, tiles.
//
// PAPER §2.1 (P133-142): overlap gamma = gamma extra layers of points around the
// owned ("green") points; the external interface ("red") points carry the
// exchange.  §3.2.2 (P292-297): local subdomain matrix + interface matrix, the
// boundary data entering through an SpMV.  Alg. 1 "initialization_and_setup"
// (P233-237), untimed (P229-231).  Readings R1 (graph-hop overlap), R4
// (exchange carries (Omega_p \ S_p) u Gamma_p), R23 (storage / id order).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "plan_internal.h"

namespace ras {

static thread_local std::string g_tls_err;
void set_tls_error(const std::string& msg) { g_tls_err = msg; }
const std::string& tls_error() { return g_tls_err; }

static constexpr int kSlice = 32;

static Fail fail(ras_status st, const std::string& m) { return Fail{st, m}; }

// Accessor for the borrowed CSR window with validation of every row touched.
struct Window {
  const ras_plan* pl;
  const int64_t* rowp(int64_t g, int64_t* len) const {
    int64_t i = g - pl->row_begin;
    if (i < 0 || i >= pl->nrows_win)
      throw fail(RAS_EINVAL, "row " + std::to_string(g) + " of an Omega_p is outside the CSR row window [" +
                                 std::to_string(pl->row_begin) + ", " + std::to_string(pl->row_begin + pl->nrows_win) +
                                 ")");
    int64_t a = pl->A_ptr[i], b = pl->A_ptr[i + 1];
    *len = b - a;
    return pl->A_ptr + i;
  }
};

static void check_rows(const ras_plan* pl) {
  // structural validation of the whole window (sorted, in range)
  if (pl->A_ptr[0] != 0) throw fail(RAS_EINVAL, "row_ptr[0] must be 0");
  for (int64_t i = 0; i < pl->nrows_win; ++i) {
    int64_t a = pl->A_ptr[i], b = pl->A_ptr[i + 1];
    if (b < a) throw fail(RAS_EINVAL, "row_ptr not monotone at row " + std::to_string(pl->row_begin + i));
    int64_t prev = -1;
    for (int64_t k = a; k < b; ++k) {
      int64_t c = pl->A_col[k];
      if (c < 0 || c >= pl->n)
        throw fail(RAS_EINVAL, "column " + std::to_string(c) + " out of range in row " + std::to_string(pl->row_begin + i));
      if (c <= prev)
        throw fail(RAS_EINVAL, "columns not strictly increasing in row " + std::to_string(pl->row_begin + i));
      prev = c;
    }
  }
}

static void build_phase1(ras_plan* pl, const ras_partition* part, const PlanDeviceHook* hook) {
  const int64_t n = pl->n;
  const int32_t P = pl->P;
  // ---- subdomain -> rank ----
  pl->sub_to_rank.resize(P);
  for (int32_t p = 0; p < P; ++p) {
    int32_t r = part->sub_to_rank ? part->sub_to_rank[p] : (int32_t)(((int64_t)p * pl->world) / P);
    if (r < 0 || r >= pl->world) throw fail(RAS_EINVAL, "sub_to_rank[" + std::to_string(p) + "] out of range");
    pl->sub_to_rank[p] = r;
  }
  // ---- owned sets (scan owner once) ----
  std::vector<int64_t> count(P, 0);
  std::vector<int32_t> local_of(P, -1);
  for (int32_t p = 0; p < P; ++p)
    if (pl->sub_to_rank[p] == pl->rank) {
      local_of[p] = (int32_t)pl->subs.size();
      pl->subs.emplace_back();
      pl->subs.back().p = p;
    }
  if (pl->subs.empty()) throw fail(RAS_EINVAL, "rank " + std::to_string(pl->rank) + " has no subdomain");
  std::vector<std::vector<int64_t>> owned_sets(pl->subs.size());
  for (int64_t g = 0; g < n; ++g) {
    int32_t p = part->owner[g];
    if (p < 0 || p >= P)
      throw fail(RAS_EINVAL, "owner[" + std::to_string(g) + "] = " + std::to_string(p) + " outside [0," +
                                 std::to_string(P) + ")");
    ++count[p];
    if (local_of[p] >= 0) owned_sets[local_of[p]].push_back(g);
  }
  for (int32_t p = 0; p < P; ++p)
    if (count[p] == 0) throw fail(RAS_EINVAL, "subdomain " + std::to_string(p) + " is empty");

  if (hook) {
    // overlap sets, owned / halo slots, receive counts built on the device
    // (setup_dev.cu); the host keeps only the bookkeeping below
    ras_status st = hook->fn(hook->user, pl, part);
    if (st != RAS_OK) throw fail(st, tls_error());
    if (pl->n_own > INT32_MAX / 2) throw fail(RAS_EINVAL, "too many owned rows on one rank for int32 slots");
    pl->send_gid.assign(pl->world, {});
    pl->send_slot.assign(pl->world, {});
    pl->send_remote_off.assign(pl->world, 0);
    pl->send_set.assign(pl->world, 0);
    pl->send_set[pl->rank] = 1;
    return;
  }
  // ---- gamma-hop BFS per local subdomain (R1, P136-140) ----
  Window W{pl};
  std::vector<int32_t> mark(n, -1), gmark(n, -1);
  const int32_t nl = (int32_t)pl->subs.size();
  for (int32_t lp = 0; lp < nl; ++lp) {
    auto& S = pl->subs[lp];
    std::vector<int64_t>& own = owned_sets[lp];
    std::vector<int64_t> all = own;
    for (int64_t g : own) mark[g] = lp;
    std::vector<int64_t> frontier = own, next;
    for (int32_t l = 0; l < pl->gamma && !frontier.empty(); ++l) {
      next.clear();
      for (int64_t g : frontier) {
        int64_t len;
        const int64_t* rp = W.rowp(g, &len);
        for (int64_t k = rp[0]; k < rp[0] + len; ++k) {
          int64_t c = pl->A_col[k];
          if (mark[c] != lp) {
            mark[c] = lp;
            next.push_back(c);
          }
        }
      }
      all.insert(all.end(), next.begin(), next.end());
      frontier.swap(next);
    }
    std::sort(all.begin(), all.end());
    S.omega = std::move(all);
    S.owned.resize(S.omega.size());
    for (size_t i = 0; i < S.omega.size(); ++i) S.owned[i] = part->owner[S.omega[i]] == S.p;
    // ghosts: neighbours of Omega_p outside Omega_p (P140-142)
    for (int64_t g : S.omega) {
      int64_t len;
      const int64_t* rp = W.rowp(g, &len);
      for (int64_t k = rp[0]; k < rp[0] + len; ++k) {
        int64_t c = pl->A_col[k];
        if (mark[c] != lp && gmark[c] != lp) {
          gmark[c] = lp;
          S.ghosts.push_back(c);
        }
      }
    }
    std::sort(S.ghosts.begin(), S.ghosts.end());
  }
  std::vector<int32_t>().swap(gmark);

  // ---- owned slots: local subdomains ascending, S_p ascending ----
  pl->slot.assign(n, -1);
  int64_t off = 0;
  for (auto& S : pl->subs) {
    S.own_off = off;
    S.nown = 0;
    for (size_t i = 0; i < S.omega.size(); ++i)
      if (S.owned[i]) {
        pl->slot[S.omega[i]] = (int32_t)(off + S.nown);
        pl->own_gid.push_back(S.omega[i]);
        ++S.nown;
      }
    off += S.nown;
  }
  pl->n_own = off;
  if (pl->n_own > INT32_MAX / 2) throw fail(RAS_EINVAL, "too many owned rows on one rank for int32 slots");

  // ---- halo: values of need_p owned by other ranks, deduped (R4) ----
  std::vector<int64_t> halo;
  std::vector<uint8_t> hmark(n, 0);
  auto add = [&](int64_t g) {
    int32_t q = pl->sub_to_rank[part->owner[g]];
    if (q != pl->rank && !hmark[g]) {
      hmark[g] = 1;
      halo.push_back(g);
    }
  };
  for (auto& S : pl->subs) {
    std::vector<int32_t> src;  // owner subdomain of every value of need_p = (Omega_p \ S_p) u Gamma_p
    for (size_t i = 0; i < S.omega.size(); ++i)
      if (!S.owned[i]) {
        add(S.omega[i]);
        src.push_back(part->owner[S.omega[i]]);
      }
    for (int64_t g : S.ghosts) {
      add(g);
      src.push_back(part->owner[g]);
    }
    std::sort(src.begin(), src.end());
    for (size_t i = 0; i < src.size();) {  // run lengths: neighbour subdomains and receive counts (Fig. 2)
      size_t j = i;
      while (j < src.size() && src[j] == src[i]) ++j;
      S.nbr_subs.push_back(src[i]);
      S.nbr_cnt.push_back((int64_t)(j - i));
      i = j;
    }
  }
  std::vector<uint8_t>().swap(hmark);
  std::sort(halo.begin(), halo.end(), [&](int64_t a, int64_t b) {
    int32_t ra = pl->sub_to_rank[part->owner[a]], rb = pl->sub_to_rank[part->owner[b]];
    return ra != rb ? ra < rb : a < b;
  });
  pl->halo_off.assign(pl->world + 1, 0);
  for (int64_t g : halo) pl->halo_off[pl->sub_to_rank[part->owner[g]] + 1]++;
  for (int32_t r = 0; r < pl->world; ++r) pl->halo_off[r + 1] += pl->halo_off[r];
  pl->n_halo = (int64_t)halo.size();
  for (int64_t i = 0; i < pl->n_halo; ++i) pl->slot[halo[i]] = (int32_t)(pl->n_own + i);
  pl->halo_gid = std::move(halo);

  pl->send_gid.assign(pl->world, {});
  pl->send_slot.assign(pl->world, {});
  pl->send_remote_off.assign(pl->world, 0);
  pl->send_set.assign(pl->world, 0);
  pl->send_set[pl->rank] = 1;
}

static void build_finalize(ras_plan* pl) {
  for (int32_t r = 0; r < pl->world; ++r)
    if (!pl->send_set[r])
      throw fail(RAS_ESTATE, "ras_plan_finalize: send list for rank " + std::to_string(r) + " not set");
  Window W{pl};
  const int64_t n = pl->n;
  const int T = pl->tile_rows;
  // row space
  int64_t roff = 0, toff = 0;
  for (auto& S : pl->subs) {
    S.row_off = roff;
    S.nrows = (int64_t)S.omega.size();
    S.nrows_pad = (S.nrows + kSlice - 1) / kSlice * kSlice;
    if (S.nrows_pad == 0) S.nrows_pad = kSlice;
    S.tile_begin = toff;
    S.ntiles = (S.nrows_pad + T - 1) / T;
    roff += S.nrows_pad;
    toff += S.ntiles;
  }
  pl->rows_pad = roff;
  if (roff >= INT32_MAX) throw fail(RAS_EINVAL, "row space exceeds int32 on one rank");
  pl->rows_local = 0;
  for (auto& S : pl->subs) pl->rows_local += S.nrows;
  const int64_t nsl = roff / kSlice;
  pl->b_loc.assign(roff, 0.0);
  pl->diag.assign(roff, 1.0);
  pl->own_slot.assign(roff, -1);
  pl->self_slot.assign(roff, 0);
  pl->slice_sub.assign(nsl, 0);
  pl->R_sptr.assign(nsl + 1, 0);
  pl->L_sptr.assign(nsl + 1, 0);
  pl->Ap_ptr.assign(roff + 1, 0);
  pl->tile_sub.clear();
  pl->tile_row0.clear();
  pl->tile_nrows.clear();

  std::vector<int32_t> mark(n, -1), pos(n, -1);
  pl->b2_global_local = 0.0;
  pl->nnz_residual = pl->nnz_local = 0;
  const int32_t nl = (int32_t)pl->subs.size();
  for (int32_t lp = 0; lp < nl; ++lp) {
    auto& S = pl->subs[lp];
    for (int64_t i = 0; i < S.nrows; ++i) {
      mark[S.omega[i]] = lp;
      pos[S.omega[i]] = (int32_t)i;
    }
    for (int64_t t = 0; t < S.ntiles; ++t) {
      pl->tile_sub.push_back(lp);
      pl->tile_row0.push_back(S.row_off + t * T);
      pl->tile_nrows.push_back((int32_t)std::min<int64_t>(T, S.nrows_pad - t * T));
    }
    S.b2 = S.b2_owned = 0.0;
    // pass 1: per-row data, slice widths
    for (int64_t s0 = 0; s0 < S.nrows_pad; s0 += kSlice) {
      const int64_t sl = (S.row_off + s0) / kSlice;
      pl->slice_sub[sl] = lp;
      int64_t wR = 0, wL = 0;
      for (int64_t i = s0; i < s0 + kSlice && i < S.nrows; ++i) {
        const int64_t g = S.omega[i];
        const int64_t row = S.row_off + i;
        int64_t len;
        const int64_t* rp = W.rowp(g, &len);
        int64_t nl_ = 0;
        bool has_diag = false;
        double outside = 0.0;  // sum of |a_ij| over the columns outside Omega_p (ascending j)
        for (int64_t k = rp[0]; k < rp[0] + len; ++k) {
          int64_t c = pl->A_col[k];
          if (mark[c] == lp) {
            if (c == g) {
              has_diag = true;
              pl->diag[row] = pl->A_val[k];
            } else {
              ++nl_;
            }
          } else {
            outside += std::fabs(pl->A_val[k]);
          }
        }
        // ORAS (R30): the local matrix's diagonal carries the Robin term; R keeps A
        if (pl->robin != 0.0) pl->diag[row] = pl->diag[row] - pl->robin * outside;
        if (!has_diag || !(pl->diag[row] > 0.0))
          throw fail(RAS_ENOTSPD, "subdomain " + std::to_string(S.p) + ": non-positive or missing diagonal at row " +
                                      std::to_string(g));
        wR = std::max(wR, len);
        wL = std::max(wL, nl_);
        const double bv = pl->b_win ? pl->b_win[g - pl->row_begin] : 0.0;
        pl->b_loc[row] = bv;
        S.b2 += bv * bv;
        if (S.owned[i]) {
          S.b2_owned += bv * bv;
          pl->own_slot[row] = pl->slot[g];
        }
        pl->self_slot[row] = pl->slot[g];
        pl->nnz_residual += len;
        pl->nnz_local += nl_ + 1;
      }
      pl->R_sptr[sl + 1] = wR * kSlice;
      pl->L_sptr[sl + 1] = wL * kSlice;
    }
    pl->b2_global_local += S.b2_owned;
  }
  for (int64_t s = 0; s < nsl; ++s) {
    pl->R_sptr[s + 1] += pl->R_sptr[s];
    pl->L_sptr[s + 1] += pl->L_sptr[s];
  }
  pl->R_col.assign(pl->R_sptr[nsl], 0);
  pl->R_val.assign(pl->R_sptr[nsl], 0.0);
  pl->L_col.assign(pl->L_sptr[nsl], 0);
  pl->L_val.assign(pl->L_sptr[nsl], 0.0);
  pl->Ap_col.clear();
  pl->Ap_val.clear();
  pl->Ap_col.reserve(pl->nnz_local + (roff - pl->rows_local));
  pl->Ap_val.reserve(pl->nnz_local + (roff - pl->rows_local));
  // pass 2: fill
  for (int32_t lp = 0; lp < nl; ++lp) {
    auto& S = pl->subs[lp];
    for (int64_t i = 0; i < S.nrows; ++i) {
      mark[S.omega[i]] = lp;
      pos[S.omega[i]] = (int32_t)i;
    }
    for (int64_t i = 0; i < S.nrows_pad; ++i) {
      const int64_t row = S.row_off + i;
      const int64_t sl = row / kSlice, lane = row % kSlice;
      const int64_t wR = (pl->R_sptr[sl + 1] - pl->R_sptr[sl]) / kSlice;
      const int64_t wL = (pl->L_sptr[sl + 1] - pl->L_sptr[sl]) / kSlice;
      int64_t kR = 0, kL = 0;
      if (i < S.nrows) {
        const int64_t g = S.omega[i];
        int64_t len;
        const int64_t* rp = W.rowp(g, &len);
        for (int64_t k = rp[0]; k < rp[0] + len; ++k) {
          const int64_t c = pl->A_col[k];
          const double v = pl->A_val[k];
          const int64_t eR = pl->R_sptr[sl] + kR * kSlice + lane;
          pl->R_col[eR] = pl->slot[c];
          pl->R_val[eR] = v;
          ++kR;
          if (mark[c] == lp) {
            pl->Ap_col.push_back(pos[c]);
            pl->Ap_val.push_back(c == g ? pl->diag[row] : v);  // diagonal of A~_p (R30)
            if (c != g) {
              const int64_t eL = pl->L_sptr[sl] + kL * kSlice + lane;
              pl->L_col[eL] = (int32_t)(S.row_off + pos[c]);
              pl->L_val[eL] = v;
              ++kL;
            }
          }
        }
      } else {
        pl->Ap_col.push_back((int32_t)i);  // padding row: identity
        pl->Ap_val.push_back(1.0);
      }
      pl->Ap_ptr[row + 1] = (int64_t)pl->Ap_col.size();
      for (; kR < wR; ++kR) {  // SELL padding: zero value, the row's own slot
        const int64_t eR = pl->R_sptr[sl] + kR * kSlice + lane;
        pl->R_col[eR] = pl->self_slot[row];
        pl->R_val[eR] = 0.0;
      }
      for (; kL < wL; ++kL) {
        const int64_t eL = pl->L_sptr[sl] + kL * kSlice + lane;
        pl->L_col[eL] = (int32_t)row;
        pl->L_val[eL] = 0.0;
      }
    }
  }
  // per tile: the span of local-matrix columns it reads (its rows included),
  // staged in shared memory by the SpMV when it fits (kernels.cuh kStageMax)
  pl->tile_cmin.assign(pl->tile_row0.size(), 0);
  pl->tile_clen.assign(pl->tile_row0.size(), -1);
  for (size_t t = 0; t < pl->tile_row0.size(); ++t) {
    const int64_t r0 = pl->tile_row0[t], r1 = pl->tile_row0[t] + pl->tile_nrows[t] - 1;
    int64_t lo = r0, hi = r1;
    for (int64_t sl = r0 / kSlice; sl <= r1 / kSlice; ++sl)
      for (int64_t e = pl->L_sptr[sl]; e < pl->L_sptr[sl + 1]; ++e) {
        lo = std::min<int64_t>(lo, pl->L_col[e]);
        hi = std::max<int64_t>(hi, pl->L_col[e]);
      }
    pl->tile_cmin[t] = (int32_t)lo;
    if (hi - lo + 1 <= pl->stage_max) pl->tile_clen[t] = (int32_t)(hi - lo + 1);
  }
  build_zformat(pl);
  pl->finalized = true;
}

}  // namespace ras

using ras::Fail;

extern "C" {

ras_status ras_plan_build(ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part,
                          int32_t overlap, int32_t rank, int32_t world) {
  return ras::plan_build_ex(out, A, b, part, overlap, rank, world, nullptr);
}

}  // extern "C"

namespace ras {
ras_status plan_build_ex(ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part, int32_t overlap,
                         int32_t rank, int32_t world, const PlanDeviceHook* hook) {
  if (!out) {
    ras::set_tls_error("ras_plan_build: out is NULL");
    return RAS_EINVAL;
  }
  *out = nullptr;
  ras_plan* pl = nullptr;
  try {
    if (!A || !part || !part->owner || !A->row_ptr || (A->nrows > 0 && (!A->col_idx || !A->val)))
      throw Fail{RAS_EINVAL, "NULL matrix / partition argument"};
    if (A->n <= 0 || A->n >= INT32_MAX) throw Fail{RAS_EINVAL, "n must be in [1, 2^31-1)"};
    if (A->row_begin < 0 || A->nrows < 0 || A->row_begin + A->nrows > A->n)
      throw Fail{RAS_EINVAL, "row window outside [0, n)"};
    if (overlap < 0) throw Fail{RAS_EINVAL, "overlap must be >= 0"};
    if (part->num_subdomains < 1) throw Fail{RAS_EINVAL, "num_subdomains must be >= 1"};
    if (world < 1 || rank < 0 || rank >= world) throw Fail{RAS_EINVAL, "bad rank / world"};
    pl = new ras_plan();
    pl->n = A->n;
    pl->P = part->num_subdomains;
    pl->rank = rank;
    pl->world = world;
    pl->gamma = overlap;
    pl->row_begin = A->row_begin;
    pl->nrows_win = A->nrows;
    pl->A_ptr = A->row_ptr;
    pl->A_col = A->col_idx;
    pl->A_val = A->val;
    pl->b_win = b;
    ras::check_rows(pl);
    ras::build_phase1(pl, part, hook);
    *out = pl;
    return RAS_OK;
  } catch (const Fail& f) {
    delete pl;
    ras::set_tls_error(f.msg);
    return f.st;
  } catch (const std::bad_alloc&) {
    delete pl;
    ras::set_tls_error("ras_plan_build: out of host memory");
    return RAS_ENOMEM;
  }
}

}  // namespace ras

extern "C" {

ras_status ras_plan_get_info(const ras_plan* pl, ras_plan_info* info) {
  if (!pl || !info) return RAS_EINVAL;
  std::memset(info, 0, sizeof(*info));
  info->n = pl->n;
  info->num_subdomains = pl->P;
  info->rank = pl->rank;
  info->world = pl->world;
  info->overlap = pl->gamma;
  info->local_subdomains = (int32_t)pl->subs.size();
  info->tile_rows = pl->tile_rows;
  info->n_own = pl->n_own;
  info->n_halo = pl->n_halo;
  int64_t rl = 0;
  for (auto& S : pl->subs) rl += (int64_t)S.omega.size();
  info->rows_local = rl;
  info->rows_padded = pl->rows_pad;
  info->nnz_residual = pl->nnz_residual;
  info->nnz_local = pl->nnz_local;
  info->sell_residual = pl->R_sptr.empty() ? 0 : pl->R_sptr.back();
  info->sell_local = pl->L_sptr.empty() ? 0 : pl->L_sptr.back();
  info->ntiles = (int64_t)pl->tile_sub.size();
  info->finalized = pl->finalized;
  info->z_format = pl->z_ok ? 1 : 0;
  return RAS_OK;
}

ras_status ras_plan_halo_request(const ras_plan* pl, int32_t src, int64_t* count, int64_t* gids_out,
                                 int64_t* halo_offset) {
  if (!pl || !count || src < 0 || src >= pl->world) return RAS_EINVAL;
  const int64_t a = pl->halo_off[src], b = pl->halo_off[src + 1];
  *count = b - a;
  if (halo_offset) *halo_offset = a;
  if (gids_out)
    for (int64_t i = a; i < b; ++i) gids_out[i - a] = pl->halo_gid[i];
  return RAS_OK;
}

ras_status ras_plan_set_send(ras_plan* pl, int32_t dst, int64_t count, const int64_t* gids, int64_t remote_offset) {
  if (!pl || dst < 0 || dst >= pl->world || count < 0 || (count > 0 && !gids)) {
    ras::set_tls_error("ras_plan_set_send: bad argument");
    return RAS_EINVAL;
  }
  if (dst == pl->rank && count != 0) {
    ras::set_tls_error("ras_plan_set_send: a rank never sends to itself");
    return RAS_EINVAL;
  }
  std::vector<int64_t> g(gids, gids + count);
  std::vector<int32_t> s(count);
  for (int64_t i = 0; i < count; ++i) {
    if (g[i] < 0 || g[i] >= pl->n || pl->slot[g[i]] < 0 || pl->slot[g[i]] >= pl->n_own) {
      ras::set_tls_error("ras_plan_set_send: rank " + std::to_string(dst) + " requested global id " +
                         std::to_string(g[i]) + " which rank " + std::to_string(pl->rank) + " does not own");
      return RAS_EINVAL;
    }
    s[i] = pl->slot[g[i]];
  }
  pl->send_gid[dst] = std::move(g);
  pl->send_slot[dst] = std::move(s);
  pl->send_remote_off[dst] = remote_offset;
  pl->send_set[dst] = 1;
  return RAS_OK;
}

ras_status ras_plan_finalize(ras_plan* pl) {
  if (!pl) return RAS_EINVAL;
  try {
    ras::build_finalize(pl);
    return RAS_OK;
  } catch (const Fail& f) {
    ras::set_tls_error(f.msg);
    return f.st;
  } catch (const std::bad_alloc&) {
    ras::set_tls_error("ras_plan_finalize: out of host memory");
    return RAS_ENOMEM;
  }
}

ras_status ras_plan_subdomain(const ras_plan* pl, int32_t li, int32_t* p_out, int64_t* nomega, int64_t* omega_out,
                              uint8_t* owned_out, int64_t* nghost, int64_t* ghosts_out) {
  if (!pl || li < 0 || li >= (int32_t)pl->subs.size()) return RAS_EINVAL;
  const auto& S = pl->subs[li];
  if (p_out) *p_out = S.p;
  if (nomega) *nomega = (int64_t)S.omega.size();
  if (nghost) *nghost = (int64_t)S.ghosts.size();
  if (omega_out) std::copy(S.omega.begin(), S.omega.end(), omega_out);
  if (owned_out) std::copy(S.owned.begin(), S.owned.end(), owned_out);
  if (ghosts_out) std::copy(S.ghosts.begin(), S.ghosts.end(), ghosts_out);
  return RAS_OK;
}

ras_status ras_plan_maps(const ras_plan* pl, int32_t li, int32_t* restrict_slot, int32_t* prolong_slot,
                         int32_t* ghost_slot) {
  if (!pl || li < 0 || li >= (int32_t)pl->subs.size()) return RAS_EINVAL;
  const auto& S = pl->subs[li];
  for (size_t i = 0; i < S.omega.size(); ++i) {
    const int32_t sl = pl->slot[S.omega[i]];
    if (restrict_slot) restrict_slot[i] = sl;
    if (prolong_slot) prolong_slot[i] = S.owned[i] ? sl : -1;
  }
  if (ghost_slot)
    for (size_t i = 0; i < S.ghosts.size(); ++i) ghost_slot[i] = pl->slot[S.ghosts[i]];
  return RAS_OK;
}

ras_status ras_plan_send_list(const ras_plan* pl, int32_t dst, int64_t* count, int64_t* gids_out, int32_t* slots_out,
                              int64_t* remote_offset) {
  if (!pl || !count || dst < 0 || dst >= pl->world) return RAS_EINVAL;
  *count = (int64_t)pl->send_gid[dst].size();
  if (remote_offset) *remote_offset = pl->send_remote_off[dst];
  if (gids_out) std::copy(pl->send_gid[dst].begin(), pl->send_gid[dst].end(), gids_out);
  if (slots_out) std::copy(pl->send_slot[dst].begin(), pl->send_slot[dst].end(), slots_out);
  return RAS_OK;
}

ras_status ras_plan_storage_gids(const ras_plan* pl, int64_t* own_gids, int64_t* halo_gids) {
  if (!pl) return RAS_EINVAL;
  if (own_gids) std::copy(pl->own_gid.begin(), pl->own_gid.end(), own_gids);
  if (halo_gids) std::copy(pl->halo_gid.begin(), pl->halo_gid.end(), halo_gids);
  return RAS_OK;
}

ras_status ras_plan_band_cholesky(const ras_plan* pl, int32_t lp, int64_t* n, int32_t* bw, double* L_out) {
  if (!pl || !n || !bw || !pl->finalized || lp < 0 || lp >= (int32_t)pl->subs.size()) return RAS_EINVAL;
  try {
    ras_plan one = *pl;  // factor just this subdomain (copy of the plan's arrays; debug ABI)
    one.subs.assign(1, pl->subs[lp]);
    ras::BandHost H;
    ras::build_band_cholesky(&one, H);
    *n = pl->subs[lp].nrows_pad;
    *bw = H.bw[0];
    if (L_out) std::copy(H.L.begin(), H.L.end(), L_out);
    return RAS_OK;
  } catch (const Fail& f) {
    ras::set_tls_error(f.msg);
    return f.st;
  }
}

ras_status ras_plan_set_robin(ras_plan* pl, double robin) {
  if (!pl || pl->finalized || !(robin >= 0.0 && robin < 1.0)) return RAS_EINVAL;
  pl->robin = robin;
  return RAS_OK;
}

ras_status ras_plan_comm_pattern(const ras_plan* pl, int64_t* counts) {
  if (!pl || !counts) return RAS_EINVAL;
  const size_t P = (size_t)pl->P;
  std::fill(counts, counts + P * P, (int64_t)0);
  for (const auto& S : pl->subs)
    for (size_t k = 0; k < S.nbr_subs.size(); ++k) counts[(size_t)S.p * P + S.nbr_subs[k]] = S.nbr_cnt[k];
  return RAS_OK;
}

void ras_plan_free(ras_plan* pl) { delete pl; }

ras_status ras_partition_regular(int32_t nx, int32_t ny, int32_t nz, int32_t px, int32_t py, int32_t pz,
                                 int32_t* owner_out) {
  // R23 / P277-286: blocks per axis differ by <= 1, earlier blocks larger.
  if (!owner_out || nx < 1 || ny < 1 || nz < 1 || px < 1 || py < 1 || pz < 1 || px > nx || py > ny || pz > nz) {
    ras::set_tls_error("ras_partition_regular: every axis needs 1 <= blocks <= cells");
    return RAS_EINVAL;
  }
  auto axis = [](int32_t n, int32_t p) {
    std::vector<int32_t> b(n);
    const int32_t q = n / p, rem = n % p;
    int32_t c = 0;
    for (int32_t k = 0; k < p; ++k)
      for (int32_t j = 0; j < q + (k < rem ? 1 : 0); ++j) b[c++] = k;
    return b;
  };
  const auto bx = axis(nx, px), by = axis(ny, py), bz = axis(nz, pz);
  int64_t g = 0;
  for (int32_t z = 0; z < nz; ++z)
    for (int32_t y = 0; y < ny; ++y)
      for (int32_t x = 0; x < nx; ++x) owner_out[g++] = (bz[z] * py + by[y]) * px + bx[x];
  return RAS_OK;
}

}  // extern "C"
