// Compressed, lane-packed SELL-32 ("SELL-Z") of the residual and local
// matrices: the same entries as the plain SELL-32, stored with fewer bytes and
// packed so that a thread fetches all entries of its row with one vector load.
//
//  * width: every slice padded to one width Wp in {4, 8} (the matrix's widest
//    slice rounded up; wider matrices keep the plain format);
//  * values: dictionary coded (CSR-VI style) — one uint8 code per entry into a
//    table of <= 256 distinct FP64 values shared by the residual matrix, the
//    local off-diagonal matrix and the diagonal (padding entries code 0.0);
//  * columns: per (slice, k) an int32 base (the smallest column of the 32 rows)
//    plus a uint16 offset per entry; a (slice, k) group spanning more than
//    65535 columns keeps its 32 int32 columns in `wide` (base = -(group) - 1);
//  * packing: entry k of lane l of slice s at (s*32 + l)*Wp + k, so lane l reads
//    its Wp codes as one 4/8-byte load and its Wp offsets as one 8/16-byte load
//    and a warp's loads are contiguous.
// Decoding is exact (table[code] is the original double, base + offset the
// original column), so results are bitwise those of the plain SELL path.
#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "plan_internal.h"

namespace ras {

namespace {

// Value dictionary keyed by the bit pattern (exact; -0.0 != 0.0).  Matrices
// that fit have few distinct values, so a linear scan with a last-hit cache is
// faster than hashing; the scan length is capped by the 256-entry limit.
struct Coder {
  std::vector<uint64_t> bits;
  std::vector<double> table;
  size_t last = 0;
  bool enc(double v, uint8_t* out) {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    if (last < bits.size() && bits[last] == b) {
      *out = (uint8_t)last;
      return true;
    }
    for (size_t i = 0; i < bits.size(); ++i)
      if (bits[i] == b) {
        last = i;
        *out = (uint8_t)i;
        return true;
      }
    if (table.size() >= 256) return false;
    last = bits.size();
    bits.push_back(b);
    table.push_back(v);
    *out = (uint8_t)last;
    return true;
  }
};

int padded_width(const std::vector<int64_t>& sptr) {
  int64_t w = 0;
  for (size_t s = 0; s + 1 < sptr.size(); ++s) w = std::max(w, (sptr[s + 1] - sptr[s]) / 32);
  if (w <= 4) return 4;
  if (w <= 8) return 8;
  return 0;
}

// plain SELL-32 (sptr, col, val) -> packed Z arrays; false if a value does not fit the table
// self_pad: the padding column of an empty slice is the lane's own row (the
// local matrix, whose columns are row-space rows) instead of 0, so every column
// of the local matrix lies in its subdomain's rows.
bool pack(const std::vector<int64_t>& sptr, const std::vector<int32_t>& col, const std::vector<double>& val, int Wp,
          Coder& C, std::vector<uint8_t>& code, std::vector<int32_t>& kbase, std::vector<uint16_t>& d16,
          std::vector<int32_t>& wide, bool self_pad) {
  const int64_t nsl = (int64_t)sptr.size() - 1;
  code.assign((size_t)nsl * 32 * Wp, 0);
  d16.assign((size_t)nsl * 32 * Wp, 0);
  kbase.assign((size_t)nsl * Wp, 0);
  wide.clear();
  uint8_t zero;
  if (!C.enc(0.0, &zero)) return false;
  std::vector<int32_t> cg(32);
  for (int64_t s = 0; s < nsl; ++s) {
    const int64_t w = (sptr[s + 1] - sptr[s]) / 32;
    for (int k = 0; k < Wp; ++k) {
      for (int l = 0; l < 32; ++l) {
        const size_t z = ((size_t)s * 32 + l) * Wp + k;
        if (k < w) {
          const int64_t e = sptr[s] + (int64_t)k * 32 + l;
          if (!C.enc(val[e], &code[z])) return false;
          cg[l] = col[e];
        } else {
          code[z] = zero;  // padding: value 0 at a valid column (the lane's first entry, or 0 / own row)
          cg[l] = w > 0 ? col[sptr[s] + l] : self_pad ? (int32_t)(s * 32 + l) : 0;
        }
      }
      const int32_t lo = *std::min_element(cg.begin(), cg.end());
      const int32_t hi = *std::max_element(cg.begin(), cg.end());
      if ((int64_t)hi - lo > 65535) {
        kbase[(size_t)s * Wp + k] = -(int32_t)(wide.size() / 32) - 1;
        wide.insert(wide.end(), cg.begin(), cg.end());
      } else {
        kbase[(size_t)s * Wp + k] = lo;
        for (int l = 0; l < 32; ++l) d16[((size_t)s * 32 + l) * Wp + k] = (uint16_t)(cg[l] - lo);
      }
    }
  }
  return true;
}

}  // namespace

bool build_zformat(ras_plan* pl) {
  pl->z_ok = false;
  const int wR = padded_width(pl->R_sptr), wL = padded_width(pl->L_sptr);
  if (!wR || !wL) return false;
  Coder C;
  std::vector<uint8_t> rc, lc, dc(pl->diag.size());
  std::vector<int32_t> rkb, lkb, rw, lw;
  std::vector<uint16_t> rd, ld;
  if (!pack(pl->R_sptr, pl->R_col, pl->R_val, wR, C, rc, rkb, rd, rw, false)) return false;
  if (!pack(pl->L_sptr, pl->L_col, pl->L_val, wL, C, lc, lkb, ld, lw, true)) return false;
  for (size_t i = 0; i < dc.size(); ++i)
    if (!C.enc(pl->diag[i], &dc[i])) return false;
  // worth it only if the wide groups stay rare
  if (rw.size() * 8 > rc.size() || lw.size() * 8 > lc.size()) return false;
  pl->z_table = std::move(C.table);
  pl->zR_w = wR;
  pl->zL_w = wL;
  pl->R_code = std::move(rc);
  pl->L_code = std::move(lc);
  pl->D_code = std::move(dc);
  pl->R_kbase = std::move(rkb);
  pl->L_kbase = std::move(lkb);
  pl->R_d16 = std::move(rd);
  pl->L_d16 = std::move(ld);
  pl->R_wide = std::move(rw);
  pl->L_wide = std::move(lw);
  pl->z_ok = true;
  return true;
}

}  // namespace ras
