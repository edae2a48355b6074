// Asynchronous mode (PAPER §3.4 "Asynchronous Schwarz setup", P389-397) — placeholder,
// replaced by the NVLink P2P implementation.
#include "ctx.h"

namespace ras {
ras_status async_setup(ras_ctx* c) { (void)c; return RAS_OK; }
void async_free(ras_ctx* c) { (void)c; }
ras_status solve_async(ras_ctx* c, double tol, int64_t max_iters) {
  (void)tol; (void)max_iters;
  return set_err(c, RAS_ESTATE, "async mode not built yet");
}
}  // namespace ras
