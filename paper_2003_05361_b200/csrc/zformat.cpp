// Compressed SELL-32 ("SELL-Z") of the residual and local matrices: the same
// entries in the same order, stored with fewer bytes when the matrix allows it.
//
//  * values: dictionary coded (CSR-VI style) — one uint8 code per entry into a
//    table of <= 256 distinct FP64 values shared by the residual matrix, the
//    local off-diagonal matrix and the diagonal;
//  * columns: per (slice, k) column of 32 entries an int32 base (the smallest
//    column) plus a uint16 offset per entry.
// Decoding is exact (table[code] is the original double, base + offset the
// original column), so results are bitwise those of the plain SELL path.  A
// matrix that does not fit (more than 256 distinct values, or a slice column
// spanning more than 65535 indices) keeps the plain FP64 / int32 format.
#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "plan_internal.h"

namespace ras {

// Groups whose 32 columns span more than 65535 (e.g. a slice straddling the
// owned / overlap boundary of the residual matrix, whose columns then point
// into two subdomains' storage) keep their int32 columns in `wide`;
// kbase = -(wide group index) - 1 marks them.
static void encode_cols(const std::vector<int32_t>& col, std::vector<int32_t>& kbase, std::vector<uint16_t>& d16,
                        std::vector<int32_t>& wide) {
  const size_t ne = col.size();
  kbase.assign(ne / 32, 0);
  d16.assign(ne, 0);
  wide.clear();
  for (size_t g = 0; g < ne / 32; ++g) {
    int32_t lo = col[g * 32], hi = col[g * 32];
    for (int l = 1; l < 32; ++l) {
      lo = std::min(lo, col[g * 32 + l]);
      hi = std::max(hi, col[g * 32 + l]);
    }
    if ((int64_t)hi - lo > 65535) {
      kbase[g] = -(int32_t)(wide.size() / 32) - 1;
      wide.insert(wide.end(), col.begin() + g * 32, col.begin() + g * 32 + 32);
      continue;
    }
    kbase[g] = lo;
    for (int l = 0; l < 32; ++l) d16[g * 32 + l] = (uint16_t)(col[g * 32 + l] - lo);
  }
}

bool build_zformat(ras_plan* pl) {
  pl->z_ok = false;
  std::unordered_map<uint64_t, uint8_t> code;
  std::vector<double> table;
  auto enc = [&](double v, uint8_t* out) -> bool {
    uint64_t b;
    std::memcpy(&b, &v, 8);
    auto it = code.find(b);
    if (it != code.end()) {
      *out = it->second;
      return true;
    }
    if (table.size() >= 256) return false;
    code.emplace(b, (uint8_t)table.size());
    *out = (uint8_t)table.size();
    table.push_back(v);
    return true;
  };
  std::vector<uint8_t> rc(pl->R_val.size()), lc(pl->L_val.size()), dc(pl->diag.size());
  for (size_t i = 0; i < rc.size(); ++i)
    if (!enc(pl->R_val[i], &rc[i])) return false;
  for (size_t i = 0; i < lc.size(); ++i)
    if (!enc(pl->L_val[i], &lc[i])) return false;
  for (size_t i = 0; i < dc.size(); ++i)
    if (!enc(pl->diag[i], &dc[i])) return false;
  std::vector<int32_t> rkb, lkb, rw, lw;
  std::vector<uint16_t> rd, ld;
  encode_cols(pl->R_col, rkb, rd, rw);
  encode_cols(pl->L_col, lkb, ld, lw);
  // worth it only if the wide groups stay rare
  if (rw.size() * 8 > pl->R_col.size() || lw.size() * 8 > pl->L_col.size()) return false;
  pl->R_wide = std::move(rw);
  pl->L_wide = std::move(lw);
  pl->z_table = std::move(table);
  pl->R_code = std::move(rc);
  pl->L_code = std::move(lc);
  pl->D_code = std::move(dc);
  pl->R_kbase = std::move(rkb);
  pl->L_kbase = std::move(lkb);
  pl->R_d16 = std::move(rd);
  pl->L_d16 = std::move(ld);
  pl->z_ok = true;
  return true;
}

}  // namespace ras
