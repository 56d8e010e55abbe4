// One instantiation of the fused DTKP apply kernel per proof count K (-DSG_DTKP_K=K), so
// the eight variants build as separate translation units in parallel.
#include "dtkp_core.cuh"

#ifndef SG_DTKP_K
#error "compile with -DSG_DTKP_K=<1..8>"
#endif

#define SG_CAT2(a, b) a##b
#define SG_CAT(a, b) SG_CAT2(a, b)

namespace sg {
int SG_CAT(launch_apply_K, SG_DTKP_K)(const DtkpK& k, int n_blocks, cudaStream_t st) {
  return launch_apply_k<SG_DTKP_K>(k, n_blocks, st);
}
}  // namespace sg
