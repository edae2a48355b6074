/*
 * ras_plan.h — host-side setup plan of the RAS hot path (row a0 of the scope
 * table): overlap construction and every index map, computed without a GPU.
 *
 * ras_setup() builds one of these per rank and uploads it; it is exported so
 * that (i) the maps can be compared bit-exactly with the oracle's sets and
 * (ii) the multi-rank exchange plan can be exercised on CPU (gloo tests).
 * All functions here are pure host code and never touch CUDA.
 *
 * Definitions (PAPER §2.1 Fig. 1, P133-142; §3.2.2, P292-297; R1, R4):
 *   S_p       rows owned by subdomain p (owner[g] == p)
 *   Omega_p   S_p plus `overlap` breadth-first layers in the graph of A, ascending
 *   Gamma_p   rows outside Omega_p adjacent to Omega_p ("red" interface points)
 *   need_p    (Omega_p \ S_p) u Gamma_p: the owner values p must receive (R4)
 * Storage of x on a rank = [owned | halo]:
 *   owned slots: the rank's subdomains in ascending id, each S_p ascending;
 *   halo slots:  every value in need_p of a local p owned by ANOTHER rank,
 *                deduplicated, sorted by (owning rank, global id) so the values
 *                from rank r form one contiguous segment [halo_off[r], halo_off[r+1]).
 * Row space on a rank: the local subdomains' Omega_p concatenated, each padded
 * to a multiple of 32 rows (one SELL-32 slice never straddles subdomains).
 */
#ifndef RAS_PLAN_H_
#define RAS_PLAN_H_

#include "ras.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ras_plan ras_plan;

typedef struct {
  int64_t n;
  int32_t num_subdomains, rank, world, overlap, local_subdomains, tile_rows;
  int64_t n_own, n_halo;      /* storage slots */
  int64_t rows_local;         /* sum |Omega_p| over local p */
  int64_t rows_padded;        /* row space incl. padding */
  int64_t nnz_residual;       /* nnz of A's rows over all local Omega_p (incl. ghost columns) */
  int64_t nnz_local;          /* nnz of all local A_p */
  int64_t sell_residual;      /* padded SELL-32 entries, residual matrix */
  int64_t sell_local;         /* padded SELL-32 entries, local off-diagonal matrix */
  int64_t ntiles;
  int32_t finalized;
  int32_t z_format;           /* 1 = the compressed SELL-Z copy exists (dictionary values, 16-bit column offsets) */
} ras_plan_info;

/* Phase 1 (local): validate inputs, build Omega_p / Gamma_p for this rank's
 * subdomains, own and halo slots, and the halo requests per source rank.
 * b may be NULL (zeros).  Exception to the borrowing rule: A's arrays and b
 * stay borrowed until ras_plan_finalize() returns (they are not copied). */
ras_status ras_plan_build(ras_plan** out, const ras_csr* A, const double* b, const ras_partition* part,
                          int32_t overlap, int32_t rank, int32_t world);

ras_status ras_plan_get_info(const ras_plan* plan, ras_plan_info* info);

/* Values this rank needs from src_rank: *count, their global ids ascending
 * (gids_out may be NULL to query the count), and where the segment starts in
 * this rank's halo (*halo_offset, relative to the first halo slot). */
ras_status ras_plan_halo_request(const ras_plan* plan, int32_t src_rank, int64_t* count, int64_t* gids_out,
                                 int64_t* halo_offset);

/* Phase 2 (exchange result): dst_rank requested `count` values `gids` (in its
 * halo order) which land at `remote_offset` in dst_rank's halo.  Every gid must
 * be owned by this rank (else RAS_EINVAL). */
ras_status ras_plan_set_send(ras_plan* plan, int32_t dst_rank, int64_t count, const int64_t* gids,
                             int64_t remote_offset);

/* Phase 3: build the row space, SELL-32 residual / local matrices, tiles. */
ras_status ras_plan_finalize(ras_plan* plan);

/* Debug export of local subdomain `local_idx` (0..local_subdomains-1).  Pass
 * NULL arrays to query sizes first.  omega_out/owned_out: len *nomega;
 * ghosts_out: len *nghost. */
ras_status ras_plan_subdomain(const ras_plan* plan, int32_t local_idx, int32_t* p_out, int64_t* nomega,
                              int64_t* omega_out, uint8_t* owned_out, int64_t* nghost, int64_t* ghosts_out);

/* Restrict / prolong maps of local subdomain `local_idx` (len |Omega_p| each):
 * restrict_slot[i] = storage slot of Omega_p[i]'s owner value;
 * prolong_slot[i]  = owned slot of Omega_p[i] if p owns it, else -1.
 * ghost_slot (len |Gamma_p|, may be NULL) = storage slot of each ghost. */
ras_status ras_plan_maps(const ras_plan* plan, int32_t local_idx, int32_t* restrict_slot, int32_t* prolong_slot,
                         int32_t* ghost_slot);

/* Pack list towards dst_rank (after set_send): global ids and owned slots. */
ras_status ras_plan_send_list(const ras_plan* plan, int32_t dst_rank, int64_t* count, int64_t* gids_out,
                              int32_t* slots_out, int64_t* remote_offset);

/* Global ids of the owned slots (len n_own) and halo slots (len n_halo). */
ras_status ras_plan_storage_gids(const ras_plan* plan, int64_t* own_gids, int64_t* halo_gids);

/* ORAS transmission parameter of the local matrices (ras_options.robin, R30); call
 * before ras_plan_finalize.  Errors: RAS_EINVAL if robin is outside [0, 1) or the plan
 * is already finalized. */
ras_status ras_plan_set_robin(ras_plan* plan, double robin);

/* Complete banded Cholesky factor of local subdomain `local_idx`'s A_p (the direct local
 * solve, RAS_LS_CHOLESKY, NEXT f1; PAPER P311-318), as the library computes it in
 * ras_setup: on return *n = padded |Omega_p| rows, *bw = bandwidth b and, if L_out is not
 * NULL, L_out[i * (b + 1) + (j - i + b)] = L(i, j) for j in [i - b, i] (row-major lower band;
 * entries outside the matrix are 0).  Call with L_out = NULL to get the sizes.  Valid after
 * ras_plan_finalize.  Errors: RAS_EINVAL (bad index / not finalized), RAS_ENOTSPD. */
ras_status ras_plan_band_cholesky(const ras_plan* plan, int32_t local_idx, int64_t* n, int32_t* bw, double* L_out);

/* Communication pattern of the partition (PAPER §3.3 "Partitioning", Fig. 2, P257-275):
 * counts[p * P + q] = number of values subdomain p receives from subdomain q per
 * exchange, i.e. |{g in (Omega_p \ S_p) u Gamma_p : owner(g) = q}| (R4), for this
 * rank's local subdomains p; every other entry is set to 0 (sum the arrays of all
 * ranks for the full matrix).  counts: caller-owned host array of P*P int64.
 * Valid after ras_plan_build.  Errors: RAS_EINVAL on NULL arguments. */
ras_status ras_plan_comm_pattern(const ras_plan* plan, int64_t* counts);

void ras_plan_free(ras_plan* plan);

/* The plan a context was built from (borrowed; valid until ras_free). */
ras_status ras_ctx_plan(const ras_ctx* ctx, const ras_plan** out);

#ifdef __cplusplus
}
#endif

#endif /* RAS_PLAN_H_ */
