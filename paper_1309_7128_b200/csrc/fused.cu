// fused.cu — the fused hot path (placeholder until the fused kernels land).
#include "solver.h"

namespace ismgb {

struct FusedEngine {};

bool fused_supported(const Solver&) { return false; }
FusedEngine* make_fused(Solver&) { return nullptr; }
void fused_solve(Solver&, Field&, const Field&, ismg_report&, Metrics&, bool, double**) {
    fail(ISMG_ERR_INTERNAL, "fused path not available");
}
void destroy_fused(FusedEngine* e) { delete e; }

}  // namespace ismgb
