// Fused Toeplitz apply chains (DAMP) for sm_100a.
//
// A left fold of Toeplitz applies — v_i = clamp01(v_{i-1} (*) S_i), i = 1..m, where each
// step is apply(f, res, d_i) with T[s0][s1] = s0 + s1 (every Sum-N fold step) — is run as
// ONE forward and ONE backward kernel instead of m of each.  Every step computes exactly
// what k_conv_fwd / k_conv_bwd compute (same FFMA order, same clamps), so results are
// bit-identical to the per-apply path; what changes is the memory traffic and the launch
// count: the running state v_{i-1} stays in shared memory between steps, so it is never
// re-read from HBM, and the m launches (each paying launch + DRAM-latency + drain) become
// one.  The clamped intermediate states are streamed out once for the backward.
//
// Reference semantics per step: provenance.py:233-253 (gather, conj, group_disj + clamp);
// backward tensor.py:287 (clamp pass-through), :415, :240, :386-391.
//
// Mapping: lane == sample; a CTA owns 32 samples for the whole chain and its warps split
// each step's output tiles; the state is a CTA-shared ping-pong pair of [n_max][32]
// shared-memory buffers (conflict-free lane access).
#include "common.cuh"

namespace sg {

constexpr int kChainMaxSteps = 32;
constexpr int kChainWarps = 4;  // warps per CTA (one CTA per 32 samples)

struct CRows {
  const float* p;
  int64_t sr, sb;
};

struct ChainArgs {
  CRows base;                      // v_0: [n[0]][B]
  CRows filt[kChainMaxSteps];      // S_i: [KF][B]
  float* dfilt_p[kChainMaxSteps];  // grad of S_i (strided like filt, writable), backward only
  int64_t dfilt_sr[kChainMaxSteps], dfilt_sb[kChainMaxSteps];
  int n[kChainMaxSteps + 1];       // n[i] = rows of v_i
  int64_t state_off[kChainMaxSteps + 1];  // row offset of v_i in `states` (i = 1..m-1)
  int m;
  int n_max;
  int64_t B;
  float* states;  // [sum_{i=1}^{m-1} n[i]][B], clamped intermediate states
  float* out;     // [n[m]][B]
  const float* g_out;  // backward: [n[m]][B]
  float* dbase_p;      // backward: grad of v_0 (strided like base)
  int64_t dbase_sr, dbase_sb;
};

__device__ __forceinline__ void pdl_wait_c() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// CTA = 32 samples (lanes) x kChainWarps warps.  The running state of the 32 samples
// lives in a CTA-shared ping-pong pair of [n_max][32] buffers; within a step the warps
// split the output tiles (R outputs each), and one __syncthreads separates the steps.
template <int KF, int R>
__global__ void __launch_bounds__(kChainWarps * 32) k_chain_fwd(const ChainArgs a) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  pdl_wait_c();
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  float* bufA = smem + lane;
  float* bufB = bufA + (size_t)a.n_max * kWarp;
  {
    const float* q = a.base.p + b * a.base.sb;
    for (int s = warp; s < a.n[0]; s += kChainWarps) bufA[s * kWarp] = __ldg(q + (int64_t)s * a.base.sr);
  }
  __syncthreads();
  for (int i = 1; i <= a.m; ++i) {
    float f[KF];
    {
      const CRows S = a.filt[i - 1];
      const float* q = S.p + b * S.sb;
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = __ldg(q + (int64_t)j * S.sr);
    }
    const int nin = a.n[i - 1], nout = a.n[i];
    const bool last = i == a.m;
    float* gdst = last ? a.out : a.states + (size_t)a.state_off[i] * a.B;
    for (int o0 = warp * R; o0 < nout; o0 += kChainWarps * R) {
      float w[R + KF - 1];
#pragma unroll
      for (int u = 0; u < R + KF - 1; ++u) {
        const int s = o0 - (KF - 1) + u;
        w[u] = (s >= 0 && s < nin) ? bufA[s * kWarp] : 0.f;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < KF; ++j) acc = fmaf(w[r + KF - 1 - j], f[j], acc);
        const int o = o0 + r;
        if (o < nout) {
          const float v = clamp01(acc);
          if (!last) bufB[o * kWarp] = v;
          if (bval) gdst[(size_t)o * a.B + b0] = v;
        }
      }
    }
    __syncthreads();
    float* t = bufA;
    bufA = bufB;
    bufB = t;
  }
}

template <int KF, int R>
__global__ void __launch_bounds__(kChainWarps * 32) k_chain_bwd(const ChainArgs a) {
  extern __shared__ float smem[];
  __shared__ float red[kChainWarps][KF][kWarp];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  pdl_wait_c();
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  float* G = smem + lane;
  float* Gn = G + (size_t)a.n_max * kWarp;
  for (int s = warp; s < a.n[a.m]; s += kChainWarps) G[s * kWarp] = __ldg(a.g_out + (size_t)s * a.B + b);
  __syncthreads();
  for (int i = a.m; i >= 1; --i) {
    float f[KF], d2[KF];
    {
      const CRows S = a.filt[i - 1];
      const float* q = S.p + b * S.sb;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        f[j] = __ldg(q + (int64_t)j * S.sr);
        d2[j] = 0.f;
      }
    }
    const int nin = a.n[i - 1], nout = a.n[i];
    const float* prev;  // v_{i-1}: the base for i == 1, else the stored clamped state
    int64_t psr;
    if (i == 1) {
      prev = a.base.p + b * a.base.sb;
      psr = a.base.sr;
    } else {
      prev = a.states + (size_t)a.state_off[i - 1] * a.B + b;
      psr = a.B;
    }
    for (int s0 = warp * R; s0 < nin; s0 += kChainWarps * R) {
      float gw[R + KF - 1];
#pragma unroll
      for (int u = 0; u < R + KF - 1; ++u) {
        const int o = s0 + u;
        gw[u] = (o < nout) ? G[o * kWarp] : 0.f;
      }
      float pv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) pv[r] = (s0 + r < nin) ? __ldg(prev + (int64_t)(s0 + r) * psr) : 0.f;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        float acc = d2[j];
#pragma unroll
        for (int r = 0; r < R; ++r) acc = fmaf(gw[r + j], pv[r], acc);
        d2[j] = acc;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < KF; ++j) acc = fmaf(gw[r + j], f[j], acc);
        const int s = s0 + r;
        if (s < nin) {
          if (i > 1)
            Gn[s * kWarp] = acc;
          else if (bval)
            a.dbase_p[(int64_t)s * a.dbase_sr + b0 * a.dbase_sb] = acc;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KF; ++j) red[warp][j][lane] = d2[j];
    __syncthreads();
    // fixed-order reduction of the warps' dS partials; warps split the KF rows
    for (int j = warp; j < KF; j += kChainWarps) {
      float acc = red[0][j][lane];
#pragma unroll
      for (int w = 1; w < kChainWarps; ++w) acc += red[w][j][lane];
      if (bval) a.dfilt_p[i - 1][(int64_t)j * a.dfilt_sr[i - 1] + b0 * a.dfilt_sb[i - 1]] = acc;
    }
    __syncthreads();
    float* t = G;
    G = Gn;
    Gn = t;
  }
}

template <typename... KArgs>
static cudaError_t launch_chain(void (*kernel)(KArgs...), const ChainArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)2 * a.n_max * kWarp * sizeof(float);
  cudaError_t e = ensure_smem((const void*)kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(a.B, kWarp));
  cfg.blockDim = dim3(kChainWarps * kWarp);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

static int fill_args(ChainArgs& a, const sg_chain* c) {
  if (c->m < 1 || c->m > kChainMaxSteps || c->kf < 1 || c->kf > 16) return (int)cudaErrorInvalidValue;
  a.base = CRows{c->base.ptr, c->base.stride_row, c->base.stride_b};
  a.m = c->m;
  a.B = c->B;
  a.n[0] = c->n0;
  int64_t off = 0;
  int nmax = c->n0;
  for (int i = 1; i <= c->m; ++i) {
    a.n[i] = a.n[i - 1] + c->kf - 1;
    a.filt[i - 1] = CRows{c->filters[i - 1].ptr, c->filters[i - 1].stride_row, c->filters[i - 1].stride_b};
    a.state_off[i] = off;
    if (i < c->m) off += a.n[i];
    if (a.n[i] > nmax) nmax = a.n[i];
  }
  a.n_max = nmax;
  a.states = c->states;
  return 0;
}

#define SG_CHAIN_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

}  // namespace sg

using namespace sg;

extern "C" {

int64_t sg_chain_states_rows(int32_t n0, int32_t kf, int32_t m) {
  int64_t rows = 0, n = n0;
  for (int i = 1; i < m; ++i) {
    n += kf - 1;
    rows += n;
  }
  return rows;
}

int sg_chain_fwd(const sg_chain* c, float* out, sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  a.out = out;
  const size_t smem = (size_t)2 * a.n_max * kWarp * sizeof(float);
  SG_RETURN_IF(smem > 200 * 1024, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K) \
  case K: return (int)launch_chain(k_chain_fwd<K, 8>, a, st);
    SG_CHAIN_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

int sg_chain_bwd(const sg_chain* c, const float* grad_out, sg_rows grad_base, const sg_rows* grad_filters,
                 sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  a.g_out = grad_out;
  a.dbase_p = grad_base.ptr;
  a.dbase_sr = grad_base.stride_row;
  a.dbase_sb = grad_base.stride_b;
  for (int i = 0; i < c->m; ++i) {
    a.dfilt_p[i] = grad_filters[i].ptr;
    a.dfilt_sr[i] = grad_filters[i].stride_row;
    a.dfilt_sb[i] = grad_filters[i].stride_b;
  }
  const size_t smem = (size_t)2 * a.n_max * kWarp * sizeof(float);
  SG_RETURN_IF(smem > 200 * 1024, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K) \
  case K: return (int)launch_chain(k_chain_bwd<K, 8>, a, st);
    SG_CHAIN_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // extern "C"
