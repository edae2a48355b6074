// Internal definition of ras_plan (host-side setup, scope row a0).  Pure C++.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "ras.h"
#include "ras_plan.h"

namespace ras {

// thread-local message of the last failure outside a context
void set_tls_error(const std::string& msg);
const std::string& tls_error();

struct Fail {
  ras_status st;
  std::string msg;
};

// One triangular factor of every local A_p in level order (factor.cpp).
struct TriHost {
  std::vector<int32_t> rows;  // row-space rows, per subdomain, by level, ascending within a level
  std::vector<int32_t> rp;    // offsets into col/val, per position in `rows` (size rows+1)
  std::vector<int32_t> col;   // row-space column of each off-diagonal dependency
  std::vector<double> val;
  std::vector<double> diag;   // per row-space row: divisor
  std::vector<std::array<int32_t, 4>> chunk;  // {rows begin, rows end, local subdomain, level}
  std::vector<int32_t> batched;               // chunk ids ordered by (level, subdomain)
  std::vector<int32_t> sub_chunk_begin, sub_chunk_end;  // per subdomain (contiguous, level order)
  std::vector<int32_t> sub_lev_off, sub_nlev;           // per subdomain: offset into lev_nchunks
  std::vector<int32_t> lev_nchunks;                     // chunks per (subdomain, level)
  std::vector<int32_t> lev_pos;      // per subdomain: nlev + 1 level-ordered positions (level l = [pos[l], pos[l+1]))
  std::vector<int32_t> sub_pos_off;  // per subdomain: offset into lev_pos (= sub_lev_off + subdomain)
  std::vector<int32_t> sub_max_lev;  // per subdomain: rows of its largest level
  int32_t max_deps = 0;              // most dependencies of any row (ELL width of the cluster solve)
  int64_t max_levels = 0;
};

// Complete banded Cholesky factors of every local A_p (factor.cpp, NEXT f1).
struct BandHost {
  std::vector<double> L, U;    // per subdomain nrows_pad x (bw + 1), row-major (see factor.cpp)
  std::vector<int64_t> off;    // per subdomain offset into L / U (size nl + 1)
  std::vector<int32_t> bw;     // per subdomain bandwidth b
};

struct SubPlan {
  int32_t p = -1;                // global subdomain id
  std::vector<int64_t> omega;    // Omega_p ascending
  std::vector<uint8_t> owned;    // per omega row
  std::vector<int64_t> ghosts;   // Gamma_p ascending
  std::vector<int32_t> nbr_subs; // owner subdomains of need_p (ascending, != p)
  std::vector<int64_t> nbr_cnt;  // values of need_p owned by each nbr_subs entry (receive counts)
  int64_t row_off = 0, nrows = 0, nrows_pad = 0;  // row space
  int64_t own_off = 0, nown = 0;                   // owned slots
  int64_t tile_begin = 0, ntiles = 0;
  double b2 = 0.0;        // ||b~_p||^2 over Omega_p (Eq. 2)
  double b2_owned = 0.0;  // ||b||^2 over S_p
};

}  // namespace ras

// Device-side phase 1 (setup_dev.cu): fills, for every local subdomain, omega /
// owned / ghosts / nbr_subs / nbr_cnt / own_off / nown, and the rank's slot map,
// own_gid, halo_gid, halo_off, n_own, n_halo -- exactly what the host BFS of
// plan.cpp computes.  Returns a ras_status (message via set_tls_error).
namespace ras {
struct PlanDeviceHook {
  ras_status (*fn)(void* user, ras_plan* pl, const ras_partition* part);
  void* user;
};
ras_status plan_build_ex(ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part, int32_t overlap,
                         int32_t rank, int32_t world, const PlanDeviceHook* hook);
}  // namespace ras

struct ras_plan {
  int64_t n = 0;
  int32_t P = 0, rank = 0, world = 1, gamma = 0;
#ifndef RAS_RPT
#define RAS_RPT 4
#endif
  int32_t tile_rows = 256 * RAS_RPT;  // must equal ras::kTileRows (kernels.cuh)
  std::vector<int32_t> sub_to_rank;
  std::vector<ras::SubPlan> subs;  // local subdomains, ascending global id
  int64_t n_own = 0, n_halo = 0;
  std::vector<int64_t> own_gid, halo_gid;
  std::vector<int64_t> halo_off;   // world + 1 (relative to the first halo slot)
  std::vector<std::vector<int64_t>> send_gid;
  std::vector<std::vector<int32_t>> send_slot;
  std::vector<int64_t> send_remote_off;
  std::vector<uint8_t> send_set;
  bool finalized = false;

  // borrowed input window (valid from ras_plan_build until ras_plan_finalize)
  int64_t row_begin = 0, nrows_win = 0;
  const int64_t* A_ptr = nullptr;
  const int32_t* A_col = nullptr;
  const double* A_val = nullptr;
  const double* b_win = nullptr;
  std::vector<int32_t> slot;  // global id -> storage slot (-1 = not stored on this rank)

  // ---- row space (after finalize) ----
  int64_t rows_pad = 0, rows_local = 0;
  std::vector<double> b_loc, diag;
  std::vector<int32_t> own_slot;   // prolong map (-1 = overlap row / padding)
  std::vector<int32_t> self_slot;  // restrict map of the row's own value
  std::vector<int32_t> slice_sub;  // local subdomain of every 32-row slice
  // SELL-32 residual matrix [A_p | B_p] with storage-slot columns (full rows)
  std::vector<int64_t> R_sptr;
  std::vector<int32_t> R_col;
  std::vector<double> R_val;
  // SELL-32 local matrix A_p, off-diagonal part, row-space columns
  std::vector<int64_t> L_sptr;
  std::vector<int32_t> L_col;
  std::vector<double> L_val;
  // CSR of A_p (subdomain-relative columns, incl. diagonal) for factorizations
  std::vector<int64_t> Ap_ptr;   // rows_pad + 1 (padding rows: diagonal 1)
  std::vector<int32_t> Ap_col;   // subdomain-relative
  std::vector<double> Ap_val;
  int64_t nnz_residual = 0, nnz_local = 0;
  // compressed SELL-Z copies of R, L and the diagonal (zformat.cpp); z_ok = usable
  bool z_ok = false;
  int32_t zR_w = 0, zL_w = 0;  // packed widths (4 or 8)
  std::vector<double> z_table;
  std::vector<uint8_t> R_code, L_code, D_code;
  std::vector<int32_t> R_kbase, L_kbase;
  std::vector<uint16_t> R_d16, L_d16;
  std::vector<int32_t> R_wide, L_wide;  // int32 columns of the groups too wide for 16-bit offsets
  // tiles: CTA work units, never straddle subdomains
  std::vector<int32_t> tile_sub;
  std::vector<int64_t> tile_row0;
  std::vector<int32_t> tile_nrows;
  std::vector<int32_t> tile_cmin, tile_clen;  // local-matrix column span per tile (-1 = wider than stage_max)
  int32_t stage_max = 4096;                   // must equal ras::kStageMax (kernels.cuh)
  double b2_global_local = 0.0;  // sum over this rank's owned rows of b^2
  double robin = 0.0;            // ORAS: A~_p,ii = a_ii - robin * sum_{j not in Omega_p} |a_ij| (R30)
};

namespace ras {
// IC(0) (kind = RAS_LS_IC0_PCG) or ILU(0) factors of every local A_p, in level
// order: F = forward (L), B = backward (L^T or U).  Throws Fail on a pivot <= 0.
void build_factors(ras_plan* pl, int kind, TriHost& F, TriHost& B);
// Complete banded Cholesky factors (L and L^T bands) of every local A_p.  Throws Fail.
void build_band_cholesky(const ras_plan* pl, BandHost& H);
// Dictionary-coded values + base/offset columns of R, L, diag; false = not compressible.
bool build_zformat(ras_plan* pl);
}  // namespace ras
