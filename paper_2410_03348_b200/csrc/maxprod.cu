// Max-product ("max/DAMP variant") apply for sm_100a: conj = product, disj = max.
//
// The north star's kernel (1) names a max variant of the fused outer-product x segmented
// reduce.  The reference has no max provenance, so its semantics are built
// from the reference's own primitives: the conj fold is the DAMP product
// (provenance.py:236, left to right as distribution.py:267-269) and the bucket reduction is
// tensor.py's reduce(kind="max") (tensor.py:319-325): value = the maximum over the
// bucket, gradient to the FIRST maximal entry along the bucket axis.  Buckets are in
// first-derivation order (records of an output in enumeration order), so "first" is the
// earliest combination.  An empty bucket is 0 (the identity of max over probabilities).
// The optional clamp01 after the max passes gradients through, like DAMP's clamp
// (tensor.py:287).
//
// Forward: one lane = one sample, a warp walks one output's records (R rows of products
// of `arity` coalesced 128-byte row loads each) and keeps (best, first argmax).  The
// argmax record id per (output, sample) is saved for the backward, which runs per input
// row over the records that use that row (CSR by row, ascending record id): a record
// contributes g[out] * prod_{j != k} x_j only where it is its output's argmax.  Every
// gradient is a fixed-order sum (no atomics): bit-reproducible.
#include "common.cuh"

namespace sg {

constexpr int kMpWarps = 4;

struct MpIn {
  const float* p[SG_MAX_ARITY];
  int64_t sr[SG_MAX_ARITY], sb[SG_MAX_ARITY];
};

static MpIn mp_inputs(const sg_rows* in, int arity) {
  MpIn m{};
  for (int i = 0; i < arity; ++i) {
    m.p[i] = in[i].ptr;
    m.sr[i] = in[i].stride_row;
    m.sb[i] = in[i].stride_b;
  }
  return m;
}

__global__ void __launch_bounds__(kMpWarps * 32) k_maxprod_fwd(const MpIn x, int arity, const int32_t* __restrict__ seg_off,
                                                               const int32_t* __restrict__ recs, int n_out, int64_t B,
                                                               int clamp, float* __restrict__ out,
                                                               int32_t* __restrict__ argmax) {
  const int s = blockIdx.x * kMpWarps + threadIdx.y;
  const int64_t b = (int64_t)blockIdx.y * kWarp + threadIdx.x;
  if (s >= n_out || b >= B) return;
  const int c0 = __ldg(seg_off + s), c1 = __ldg(seg_off + s + 1);
  float best = 0.f;
  int arg = -1;
  for (int c = c0; c < c1; ++c) {
    const int32_t* r = recs + (size_t)c * arity;
    float v = __ldg(x.p[0] + (int64_t)__ldg(r) * x.sr[0] + b * x.sb[0]);
    for (int i = 1; i < arity; ++i) v *= __ldg(x.p[i] + (int64_t)__ldg(r + i) * x.sr[i] + b * x.sb[i]);
    if (arg < 0 || v > best) {  // strict: ties keep the first record (tensor.py:321)
      best = v;
      arg = c;
    }
  }
  out[(size_t)s * B + b] = clamp ? clamp01(best) : best;
  argmax[(size_t)s * B + b] = arg;
}

__global__ void __launch_bounds__(kMpWarps * 32) k_maxprod_bwd(const MpIn x, int arity, int k, int rows_k,
                                                               const int32_t* __restrict__ in_off,
                                                               const int32_t* __restrict__ in_recs,
                                                               const int32_t* __restrict__ recs,
                                                               const int32_t* __restrict__ rec_out, int64_t B,
                                                               const int32_t* __restrict__ argmax, const Rows g,
                                                               WRows gin) {
  const int r = blockIdx.x * kMpWarps + threadIdx.y;
  const int64_t b = (int64_t)blockIdx.y * kWarp + threadIdx.x;
  if (r >= rows_k || b >= B) return;
  float acc = 0.f;
  const int e0 = __ldg(in_off + r), e1 = __ldg(in_off + r + 1);
  for (int e = e0; e < e1; ++e) {
    const int c = __ldg(in_recs + e);
    const int s = __ldg(rec_out + c);
    if (__ldg(argmax + (size_t)s * B + b) != c) continue;
    const int32_t* rc = recs + (size_t)c * arity;
    float prod = 1.f;
    bool first = true;
    for (int i = 0; i < arity; ++i) {
      if (i == k) continue;
      const float v = __ldg(x.p[i] + (int64_t)__ldg(rc + i) * x.sr[i] + b * x.sb[i]);
      prod = first ? v : prod * v;
      first = false;
    }
    acc = fmaf(g.ld(s, b), prod, acc);
  }
  gin.st(r, b, acc);
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_maxprod_fwd(const sg_maxprod_plan* p, const sg_rows* inputs, int64_t B, int32_t clamp, float* out,
                   int32_t* argmax, sg_stream_t stream) {
  SG_RETURN_IF(p == nullptr || p->arity < 1 || p->arity > SG_MAX_ARITY, cudaErrorInvalidValue);
  if (B <= 0 || p->n_out <= 0) return 0;
  for (int i = 0; i < p->arity; ++i) SG_RETURN_IF(p->n_recs > 0 && inputs[i].ptr == nullptr, cudaErrorInvalidValue);
  const MpIn x = mp_inputs(inputs, p->arity);
  dim3 grid(ceil_div(p->n_out, kMpWarps), ceil_div(B, kWarp));
  SG_RETURN_IF(grid.y > 65535, cudaErrorInvalidValue);
  count_launch();
  k_maxprod_fwd<<<grid, dim3(kWarp, kMpWarps), 0, (cudaStream_t)stream>>>(x, p->arity, p->seg_off, p->recs, p->n_out,
                                                                            B, clamp, out, argmax);
  SG_LAUNCH_CHECK();
  return 0;
}

int sg_maxprod_bwd(const sg_maxprod_plan* p, const sg_rows* inputs, int64_t B, const int32_t* argmax,
                   sg_rows grad_out, const sg_rows* grad_in, sg_stream_t stream) {
  SG_RETURN_IF(p == nullptr || p->arity < 1 || p->arity > SG_MAX_ARITY, cudaErrorInvalidValue);
  if (B <= 0) return 0;
  const MpIn x = mp_inputs(inputs, p->arity);
  for (int k = 0; k < p->arity; ++k) {
    if (grad_in[k].ptr == nullptr || p->sizes[k] <= 0) continue;
    dim3 grid(ceil_div(p->sizes[k], kMpWarps), ceil_div(B, kWarp));
    SG_RETURN_IF(grid.y > 65535, cudaErrorInvalidValue);
    count_launch();
    k_maxprod_bwd<<<grid, dim3(kWarp, kMpWarps), 0, (cudaStream_t)stream>>>(
        x, p->arity, k, p->sizes[k], p->in_off[k], p->in_recs[k], p->recs, p->rec_out, B, argmax, rows_of(grad_out),
        wrows_of(grad_in[k]));
    SG_LAUNCH_CHECK();
  }
  return 0;
}

}  // extern "C"
