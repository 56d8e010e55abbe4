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

// ---- cp.async (LDGSTS) staging of the per-step filters: a ring of kRing slots, so the
// filters of steps i+1 .. i+kRing-2 are in flight while step i computes.
constexpr int kRing = 4;

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(kRing - 2) : "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Filter S_step (KF rows of this CTA's 32 samples) -> ring slot.
template <int KF>
__device__ __forceinline__ void stage_filter(float* ring, int slot, const CRows& S, int64_t b, int lane, int warp) {
  const float* q = S.p + b * S.sb;
  float* d = ring + (size_t)slot * KF * kWarp + lane;
  for (int j = warp; j < KF; j += kChainWarps) cp_async4(d + j * kWarp, q + (int64_t)j * S.sr);
}

__host__ __device__ constexpr int round_up(int a, int r) { return (a + r - 1) / r * r; }

// Shared-memory rows ([rows][32] fp32) of the forward / backward kernels.
__host__ __device__ inline int fwd_vrows(int kf, int r, int n_max) { return (kf - 1) + round_up(n_max, r); }
__host__ __device__ inline int bwd_grows(int kf, int r, int n_max) { return round_up(n_max, r) + r + kf; }
inline size_t fwd_smem_bytes(int kf, int r, int n_max) {
  return (size_t)(kRing * kf + 2 * fwd_vrows(kf, r, n_max)) * kWarp * sizeof(float);
}
inline size_t bwd_smem_bytes(int kf, int r, int n_max) {
  return (size_t)(kRing * kf + 2 * bwd_grows(kf, r, n_max) + 2 * kChainWarps * kf) * kWarp * sizeof(float);
}

// Forward.  CTA = 32 samples (lanes) x kChainWarps warps sharing the running state, a
// ping-pong pair of [kf-1 zero rows | state rows] shared-memory buffers.  The zero rows in
// front and the zero rows past each state's end make every window load unconditional:
// rows >= n_{i-1} of the source buffer are always exactly 0 (they are either never written
// or hold clamp01(0) from a padded tile of an earlier, shorter step).  Filters arrive
// through the cp.async ring; the only global traffic inside a step is the stores.
template <int KF, int R>
__global__ void __launch_bounds__(kChainWarps * 32) k_chain_fwd(const ChainArgs a) {
  extern __shared__ float smem[];
  constexpr int PAD = KF - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  const int vrows = fwd_vrows(KF, R, a.n_max);
  float* ring = smem;
  float* VA = ring + kRing * KF * kWarp;
  float* VB = VA + (size_t)vrows * kWarp;
  pdl_wait_c();
  for (int s = 1; s < kRing; ++s) {
    if (s <= a.m) stage_filter<KF>(ring, s % kRing, a.filt[s - 1], b, lane, warp);
    cp_commit();
  }
  {
    const float* q = a.base.p + b * a.base.sb;
    for (int r = warp; r < vrows; r += kChainWarps) {
      const int s = r - PAD;
      VA[r * kWarp + lane] = (s >= 0 && s < a.n[0]) ? __ldg(q + (int64_t)s * a.base.sr) : 0.f;
      VB[r * kWarp + lane] = 0.f;
    }
  }
  cp_wait_ring();
  __syncthreads();
  float* src = VA + PAD * kWarp + lane;
  float* dst = VB + PAD * kWarp + lane;
  for (int i = 1; i <= a.m; ++i) {
    {
      const int s = i + kRing - 1;
      if (s <= a.m) stage_filter<KF>(ring, s % kRing, a.filt[s - 1], b, lane, warp);
      cp_commit();
    }
    float f[KF];
    {
      const float* F = ring + (size_t)(i % kRing) * KF * kWarp + lane;
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = F[j * kWarp];
    }
    const int nout = a.n[i];
    const bool last = i == a.m;
    float* gdst = (last ? a.out : a.states + (size_t)a.state_off[i] * a.B) + b0;
    for (int o0 = warp * R; o0 < nout; o0 += kChainWarps * R) {
      float w[R + KF - 1];
      const float* p = src + (o0 - PAD) * kWarp;
#pragma unroll
      for (int u = 0; u < R + KF - 1; ++u) w[u] = p[u * kWarp];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < KF; ++j) acc = fmaf(w[r + KF - 1 - j], f[j], acc);
        const float v = clamp01(acc);
        const int o = o0 + r;
        if (!last) dst[o * kWarp] = v;  // padded tile rows >= nout get clamp01(0) = 0
        if (o < nout && bval) gdst[(size_t)o * a.B] = v;
      }
    }
    cp_wait_ring();
    __syncthreads();
    float* t = src;
    src = dst;
    dst = t;
  }
}

// Backward.  The upstream gradient G of the current step lives in a ping-pong pair of
// shared buffers (rows past each step's length zeroed, so windows are unconditional);
// per step every warp first issues the global loads of v_{i-1} for a chunk of its tiles
// (kChainTch tiles of R rows in flight at once, L2-prefetched one step ahead), then
// computes G_{i-1} = G_i (*)^T S_i and its dS_i partials.  dS partials are reduced across
// the warps in shared memory in fixed order (deterministic, no atomics).
constexpr int kChainTch = 4;

template <int KF, int R>
__global__ void __launch_bounds__(kChainWarps * 32) k_chain_bwd(const ChainArgs a) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  const int grows = bwd_grows(KF, R, a.n_max);
  float* ring = smem;
  float* GA = ring + kRing * KF * kWarp;
  float* GB = GA + (size_t)grows * kWarp;
  float* red = GB + (size_t)grows * kWarp;  // [2][kChainWarps][KF][32]
  pdl_wait_c();
  // bwd step t handles apply i = m - t; its filter sits in ring slot t % kRing
  for (int t = 0; t < kRing - 1; ++t) {
    if (t < a.m) stage_filter<KF>(ring, t % kRing, a.filt[a.m - 1 - t], b, lane, warp);
    cp_commit();
  }
  {
    const int nm = a.n[a.m];
    for (int r = warp; r < grows; r += kChainWarps) {
      GA[r * kWarp + lane] = r < nm ? __ldg(a.g_out + (size_t)r * a.B + b) : 0.f;
      GB[r * kWarp + lane] = 0.f;
    }
  }
  cp_wait_ring();
  __syncthreads();
  float* G = GA + lane;
  float* Gn = GB + lane;
  for (int t = 0; t < a.m; ++t) {
    const int i = a.m - t;
    {
      const int tt = t + kRing - 1;
      if (tt < a.m) stage_filter<KF>(ring, tt % kRing, a.filt[a.m - 1 - tt], b, lane, warp);
      cp_commit();
    }
    if (i > 2) {  // next step reads v_{i-2}: pull this CTA's 128-byte row segments into L2
      const float* pn = a.states + (size_t)a.state_off[i - 2] * a.B + (int64_t)blockIdx.x * kWarp;
      for (int s = threadIdx.x; s < a.n[i - 2]; s += kChainWarps * kWarp) prefetch_l2(pn + (size_t)s * a.B);
    }
    float f[KF], d2[KF];
    {
      const float* F = ring + (size_t)(t % kRing) * KF * kWarp + lane;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        f[j] = F[j * kWarp];
        d2[j] = 0.f;
      }
    }
    const int nin = a.n[i - 1];
    const float* prev;  // v_{i-1}: the base for i == 1, else the stored clamped state
    int64_t psr;
    if (i == 1) {
      prev = a.base.p + b * a.base.sb;
      psr = a.base.sr;
    } else {
      prev = a.states + (size_t)a.state_off[i - 1] * a.B + b;
      psr = a.B;
    }
    for (int c0 = warp * R; c0 < nin; c0 += kChainTch * kChainWarps * R) {
      float pv[kChainTch][R];
#pragma unroll
      for (int q = 0; q < kChainTch; ++q)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int s = c0 + q * kChainWarps * R + r;
          pv[q][r] = s < nin ? __ldg(prev + (int64_t)s * psr) : 0.f;
        }
#pragma unroll
      for (int q = 0; q < kChainTch; ++q) {
        const int s0 = c0 + q * kChainWarps * R;
        if (s0 >= nin) break;
        float gw[R + KF - 1];
#pragma unroll
        for (int u = 0; u < R + KF - 1; ++u) gw[u] = G[(s0 + u) * kWarp];
#pragma unroll
        for (int j = 0; j < KF; ++j) {
          float acc = d2[j];
#pragma unroll
          for (int r = 0; r < R; ++r) acc = fmaf(gw[r + j], pv[q][r], acc);
          d2[j] = acc;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float acc = 0.f;
#pragma unroll
          for (int j = 0; j < KF; ++j) acc = fmaf(gw[r + j], f[j], acc);
          const int s = s0 + r;
          if (i > 1)
            Gn[s * kWarp] = s < nin ? acc : 0.f;
          else if (s < nin && bval)
            a.dbase_p[(int64_t)s * a.dbase_sr + b0 * a.dbase_sb] = acc;
        }
      }
    }
    if (i > 1)  // rows past the padded tiles that the next step's windows can reach
      for (int r = round_up(nin, R) + warp; r < nin + R + KF - 1; r += kChainWarps) Gn[r * kWarp] = 0.f;
    float* rd = red + (size_t)(t & 1) * kChainWarps * KF * kWarp + lane;
#pragma unroll
    for (int j = 0; j < KF; ++j) rd[(warp * KF + j) * kWarp] = d2[j];
    cp_wait_ring();
    __syncthreads();
    for (int j = warp; j < KF; j += kChainWarps) {
      float acc = rd[j * kWarp];
#pragma unroll
      for (int w = 1; w < kChainWarps; ++w) acc += rd[(w * KF + j) * kWarp];
      if (bval) a.dfilt_p[i - 1][(int64_t)j * a.dfilt_sr[i - 1] + b0 * a.dfilt_sb[i - 1]] = acc;
    }
    float* tmp = G;
    G = Gn;
    Gn = tmp;
  }
}

template <typename... KArgs>
static cudaError_t launch_chain(void (*kernel)(KArgs...), const ChainArgs& a, size_t smem, cudaStream_t st) {
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

constexpr int kChainR = 8;                       // output rows per tile
constexpr size_t kChainSmemMax = 227 * 1024;     // sm_100 per-CTA dynamic shared memory

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
  const size_t smem = fwd_smem_bytes(c->kf, kChainR, a.n_max);
  SG_RETURN_IF(smem > kChainSmemMax, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K) \
  case K: return (int)launch_chain(k_chain_fwd<K, kChainR>, a, smem, st);
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
  const size_t smem = bwd_smem_bytes(c->kf, kChainR, a.n_max);
  SG_RETURN_IF(smem > kChainSmemMax, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K) \
  case K: return (int)launch_chain(k_chain_bwd<K, kChainR>, a, smem, st);
    SG_CHAIN_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // extern "C"
