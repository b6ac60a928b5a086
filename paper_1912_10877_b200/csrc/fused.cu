// fused.cu — tiled multi-gate engine (placeholder until the tile kernels land).
#include "program.h"

namespace qbg {

struct FusedPlan {};

bool fused_forward(const DevState&, Program&, bool) { return false; }
bool fused_backward(const DevState&, const DevState&, Program&, double*) { return false; }
bool fused_obs_apply(const DevState&, const DevState&, Observable&, double*) { return false; }
void fused_stats(const Program&, int64_t* f, int64_t* b) { *f = 0; *b = 0; }

}  // namespace qbg
