// C ABI of the fused Toeplitz apply chains (sgb200.h): picks the row-group variant of
// chain.cu (compiled once per SG_CHAIN_GROUPS) from the batch, identically for the
// forward and the backward of one chain (the states layout depends on it).
#include <cstdlib>

#include "common.cuh"

#define SG_CHAIN_VARIANT_DECL(G)                                                                                \
  namespace sg {                                                                                                \
  namespace chain_g##G {                                                                                        \
  int64_t states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B);                                          \
  int32_t max_rows(int32_t kf);                                                                                 \
  int fwd(const sg_chain* c, float* out, double* rowsum, sg_stream_t stream);                                   \
  int bwd(const sg_chain* c, const float* grad_out, sg_rows grad_base, const sg_rows* grad_filters,             \
          sg_stream_t stream);                                                                                  \
  int bwd_nll(const sg_chain* c, const int64_t* targets, const double* rowsum, const double* picked,            \
              const double* grad_loss, sg_rows grad_base, const sg_rows* grad_filters, sg_stream_t stream);     \
  }                                                                                                             \
  }
SG_CHAIN_VARIANT_DECL(4)
SG_CHAIN_VARIANT_DECL(8)
SG_CHAIN_VARIANT_DECL(16)

namespace {
// Row groups for a batch: 4 (16 samples per warp) while that still gives ~1000 warps,
// then 8 and 16 (8 / 4 samples per warp).  SG_CHAIN_G overrides (A/B measurements).
int chain_groups(int64_t B) {
  static const int forced = [] {
    const char* e = std::getenv("SG_CHAIN_G");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 4 || forced == 8 || forced == 16) return forced;
  return B >= 12288 ? 4 : B >= 6144 ? 8 : 16;
}
}  // namespace

#define SG_CHAIN_DISPATCH(B, call)                 \
  switch (chain_groups(B)) {                       \
    case 8: return sg::chain_g8::call;             \
    case 16: return sg::chain_g16::call;           \
    default: return sg::chain_g4::call;            \
  }

extern "C" {

int64_t sg_chain_states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B) {
  return sg::chain_g4::states_elems(n0, kf, m, B);  // 16 samples per warp: the largest padding
}

int32_t sg_chain_max_rows(int32_t kf) {
  return sg::chain_g4::max_rows(kf);  // the variant with the most shared memory per row
}

int sg_chain_fwd(const sg_chain* c, float* out, double* rowsum, sg_stream_t stream) {
  if (c == nullptr) return (int)cudaErrorInvalidValue;
  SG_CHAIN_DISPATCH(c->B, fwd(c, out, rowsum, stream))
}

int sg_chain_bwd(const sg_chain* c, const float* grad_out, sg_rows grad_base, const sg_rows* grad_filters,
                 sg_stream_t stream) {
  if (c == nullptr) return (int)cudaErrorInvalidValue;
  SG_CHAIN_DISPATCH(c->B, bwd(c, grad_out, grad_base, grad_filters, stream))
}

int sg_chain_bwd_nll(const sg_chain* c, const int64_t* targets, const double* rowsum, const double* picked,
                     const double* grad_loss, sg_rows grad_base, const sg_rows* grad_filters, sg_stream_t stream) {
  if (c == nullptr) return (int)cudaErrorInvalidValue;
  SG_CHAIN_DISPATCH(c->B, bwd_nll(c, targets, rowsum, picked, grad_loss, grad_base, grad_filters, stream))
}

}  // extern "C"
