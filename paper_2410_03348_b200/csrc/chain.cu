// Fused Toeplitz apply chains (DAMP) for sm_100a.
//
// A left fold of Toeplitz applies — v_i = clamp01(v_{i-1} (*) S_i), i = 1..m, where each
// step is apply(f, res, d_i) with T[s0][s1] = s0 + s1 (every Sum-N fold step) — is run as
// ONE forward and ONE backward kernel instead of m of each.  Every step computes exactly
// what k_conv_fwd / k_conv_bwd compute (same FMA order per output, same clamps), so the
// forward is bit-identical to the per-apply path; what changes is the memory traffic and
// the launch count: the running state v_{i-1} stays in shared memory between steps (it
// is never re-read from HBM) and the m launches (each paying launch + DRAM latency +
// drain) become one.  The clamped intermediate states are streamed out once for the
// backward.
//
// Reference semantics per step: provenance.py:233-253 (gather, conj, group_disj + clamp);
// backward tensor.py:287 (clamp pass-through), :415, :240, :386-391.
//
// Mapping (B200): a CTA owns 64 samples for the whole chain; lane l holds the sample PAIR
// (b0 + 2l, b0 + 2l + 1) so every multiply-add is one packed FFMA2 (fma.rn.f32x2, two
// IEEE fp32 FMAs — identical rounding to two FFMAs) and every shared-memory access is one
// conflict-free 8-byte LDS.64/STS.64 per lane.  The warps of the CTA split each step's
// output tiles (R rows each) and share the state through a ping-pong pair of
// [rows][32 lanes] float2 shared-memory buffers.  Intermediate states go to HBM in a
// CTA-blocked layout ([cta][row][64 samples]) so a tile's rows are 256-byte lines at
// immediate offsets from one base pointer.
#include "common.cuh"

namespace sg {

constexpr int kChainMaxSteps = 32;
constexpr int kChainR = 8;      // output rows per tile
constexpr int kChainNW = 8;     // warps per CTA
constexpr int kChainS = 64;     // samples per CTA (32 lanes x 2)
constexpr int kRing = 4;        // cp.async filter ring depth
#ifndef SG_CHAIN_TCH
#define SG_CHAIN_TCH 2
#endif
constexpr int kChainTch = SG_CHAIN_TCH;  // backward: tiles whose v_{i-1} loads are in flight together
constexpr size_t kChainSmemMax = 227 * 1024;
constexpr size_t kChainSmemTwo = 227 * 1024 / 2 - 1024;  // two CTAs per SM

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
  int state_off[kChainMaxSteps + 1];  // row offset of v_i inside a CTA's state block (i = 1..m-1)
  int state_rows;                  // rows of one CTA's state block
  int allf;                        // forward: all m filters fit in shared memory
  int m;
  int n_max;
  int64_t B;
  float* states;       // [ceil(B/64)][state_rows][64] clamped intermediate states
  float* out;          // [n[m]][B]
  const float* g_out;  // backward: [n[m]][B]
  float* dbase_p;      // backward: grad of v_0 (strided like base)
  int64_t dbase_sr, dbase_sb;
};

__device__ __forceinline__ void pdl_wait_c() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(kRing - 2) : "memory"); }

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 clamp01x2(float2 v) { return make_float2(clamp01(v.x), clamp01(v.y)); }

// The pair of samples a lane owns: (b0, b0 + 1); loads use clamped indices, stores are
// predicated by nv (number of valid samples of the pair: 0, 1 or 2).
struct Pair {
  int64_t b0, ba, bb;
  int nv;
};

__device__ __forceinline__ Pair lane_pair(int64_t B, int lane) {
  Pair p;
  p.b0 = (int64_t)blockIdx.x * kChainS + 2 * lane;
  const int64_t left = B - p.b0;
  p.nv = left <= 0 ? 0 : (left >= 2 ? 2 : 1);
  p.ba = p.b0 < B ? p.b0 : B - 1;
  p.bb = p.b0 + 1 < B ? p.b0 + 1 : B - 1;
  return p;
}

// Row `row` of a strided operand for the lane's two samples.
__device__ __forceinline__ float2 ld_strided(const CRows& S, const Pair& p, int64_t row) {
  return make_float2(__ldg(S.p + p.ba * S.sb + row * S.sr), __ldg(S.p + p.bb * S.sb + row * S.sr));
}

__device__ __forceinline__ void st_strided(float* base, int64_t sr, int64_t sb, const Pair& p, int64_t row, float2 v) {
  if (p.nv > 0) base[p.b0 * sb + row * sr] = v.x;
  if (p.nv > 1) base[(p.b0 + 1) * sb + row * sr] = v.y;
}

// [rows][B] contiguous row-major (out, g_out): 8-byte vector access when B is even
// (then a pair is either fully valid or fully past the end).
template <bool VEC>
__device__ __forceinline__ float2 ld_rowmajor(const float* q, const Pair& p) {  // q = row start
  if constexpr (VEC) {
    return p.nv == 2 ? __ldg(reinterpret_cast<const float2*>(q + p.b0)) : make_float2(0.f, 0.f);
  } else {
    return make_float2(__ldg(q + p.ba), __ldg(q + p.bb));
  }
}

template <bool VEC>
__device__ __forceinline__ void st_rowmajor(float* q, const Pair& p, float2 v) {
  if constexpr (VEC) {
    if (p.nv == 2) *reinterpret_cast<float2*>(q + p.b0) = v;
  } else {
    if (p.nv > 0) q[p.b0] = v.x;
    if (p.nv > 1) q[p.b0 + 1] = v.y;
  }
}

// Filter S (KF rows of this CTA's 64 samples) -> ring slot, as float2 [KF][32].
template <int KF>
__device__ __forceinline__ void stage_filter(float2* ring, int slot, const CRows& S, const Pair& p, int lane,
                                             int warp) {
  float* d = reinterpret_cast<float*>(ring + (size_t)slot * KF * kWarp + lane);
  const float* qa = S.p + p.ba * S.sb;
  const float* qb = S.p + p.bb * S.sb;
  for (int j = warp; j < KF; j += kChainNW) {
    cp_async4(d + 2 * j * kWarp, qa + (int64_t)j * S.sr);
    cp_async4(d + 2 * j * kWarp + 1, qb + (int64_t)j * S.sr);
  }
}

__host__ __device__ constexpr int round_up(int a, int r) { return (a + r - 1) / r * r; }

// Shared-memory rows ([rows][32] float2 = 256 B each) of the forward / backward kernels.
__host__ __device__ inline int fwd_vrows(int kf, int n_max) { return (kf - 1) + round_up(n_max, kChainR); }
__host__ __device__ inline int bwd_grows(int kf, int n_max) { return round_up(n_max, kChainR) + kChainR + kf; }
inline size_t fwd_smem_bytes(int kf, int n_max, int fslots = kRing) {
  return (size_t)(fslots * kf + 2 * fwd_vrows(kf, n_max)) * kWarp * sizeof(float2);
}
inline size_t bwd_smem_bytes(int kf, int n_max) {
  return (size_t)(kRing * kf + 2 * bwd_grows(kf, n_max) + kChainNW * kf) * kWarp * sizeof(float2);
}

// Forward.  Source buffer rows >= n_{i-1} are always exactly 0 (never written, or
// clamp01(0) from a padded tile of an earlier, shorter step), and kf-1 zero rows sit in
// front, so every window load is unconditional.  Filters arrive through the cp.async ring
// kRing-1 steps ahead; inside a step the only global traffic is the (streaming) stores.
template <int KF, bool VEC>
__global__ void __launch_bounds__(kChainNW * 32, 2) k_chain_fwd(const ChainArgs a) {
  extern __shared__ float2 smem2[];
  constexpr int R = kChainR, PAD = KF - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Pair pr = lane_pair(a.B, lane);
  const int vrows = fwd_vrows(KF, a.n_max);
  // all m filters staged up front when they fit (one exposed latency for the whole
  // chain), else a ring of kRing slots refilled kRing-1 steps ahead
  const int fslots = a.allf ? a.m : kRing;
  float2* ring = smem2;
  float2* VA = ring + (size_t)fslots * KF * kWarp;
  float2* VB = VA + (size_t)vrows * kWarp;
  pdl_wait_c();
  if (a.allf) {
    for (int s = 1; s <= a.m; ++s) stage_filter<KF>(ring, s - 1, a.filt[s - 1], pr, lane, warp);
    cp_commit();
  } else {
    for (int s = 1; s < kRing; ++s) {
      if (s <= a.m) stage_filter<KF>(ring, s % kRing, a.filt[s - 1], pr, lane, warp);
      cp_commit();
    }
  }
  for (int r = warp; r < vrows; r += kChainNW) {
    const int s = r - PAD;
    VA[r * kWarp + lane] = (s >= 0 && s < a.n[0]) ? ld_strided(a.base, pr, s) : make_float2(0.f, 0.f);
    VB[r * kWarp + lane] = make_float2(0.f, 0.f);
  }
  if (a.allf)
    cp_wait_all();
  else
    cp_wait_ring();
  __syncthreads();
  const float2* src = VA + PAD * kWarp + lane;
  float2* dst = VB + PAD * kWarp + lane;
  float2* sblk = reinterpret_cast<float2*>(a.states) + (size_t)blockIdx.x * a.state_rows * kWarp + lane;
  for (int i = 1; i <= a.m; ++i) {
    if (!a.allf) {
      const int s = i + kRing - 1;
      if (s <= a.m) stage_filter<KF>(ring, s % kRing, a.filt[s - 1], pr, lane, warp);
      cp_commit();
    }
    float2 f[KF];
    {
      const float2* F = ring + (size_t)(a.allf ? i - 1 : i % kRing) * KF * kWarp + lane;
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = F[j * kWarp];
    }
    const int nout = a.n[i];
    if (i < a.m) {
      float2* gst = sblk + (size_t)a.state_off[i] * kWarp;
      for (int o0 = warp * R; o0 < nout; o0 += kChainNW * R) {
        float2 w[R + KF - 1];
        const float2* p = src + (o0 - PAD) * kWarp;
#pragma unroll
        for (int u = 0; u < R + KF - 1; ++u) w[u] = p[u * kWarp];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < KF; ++j) acc = ffma2(w[r + KF - 1 - j], f[j], acc);
          const float2 v = clamp01x2(acc);
          dst[(o0 + r) * kWarp] = v;  // padded tile rows >= nout get clamp01(0) = 0
          if (o0 + r < nout) gst[(o0 + r) * kWarp] = v;
        }
      }
    } else {
      for (int o0 = warp * R; o0 < nout; o0 += kChainNW * R) {
        float2 w[R + KF - 1];
        const float2* p = src + (o0 - PAD) * kWarp;
#pragma unroll
        for (int u = 0; u < R + KF - 1; ++u) w[u] = p[u * kWarp];
        float* q = a.out + (size_t)o0 * a.B;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < KF; ++j) acc = ffma2(w[r + KF - 1 - j], f[j], acc);
          if (o0 + r < nout) st_rowmajor<VEC>(q, pr, clamp01x2(acc));
          q += a.B;
        }
      }
    }
    if (!a.allf) cp_wait_ring();
    __syncthreads();
    const float2* t = src;
    src = dst;
    dst = const_cast<float2*>(t);
  }
}

// v_{ii-1} rows c0 + q*NW*R + r (the warp's chunk of tiles) of step ii for the lane's
// pair; rows past the state's end read as 0 (they meet nonzero G rows in the dS sums).
template <int R>
__device__ __forceinline__ void load_prev(float2 (&pv)[kChainTch][R], const ChainArgs& a, const float2* sblk,
                                          const Pair& pr, int ii, int c0) {
  const int nin = a.n[ii - 1];
  const float2* pst = sblk + (size_t)a.state_off[ii - 1] * kWarp;
#pragma unroll
  for (int q = 0; q < kChainTch; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = c0 + q * kChainNW * R + r;
      if (s >= nin)
        pv[q][r] = make_float2(0.f, 0.f);
      else if (ii > 1)
        pv[q][r] = pst[s * kWarp];
      else
        pv[q][r] = ld_strided(a.base, pr, s);
    }
}

// Backward.  The upstream gradient G of the current step lives in a ping-pong pair of
// shared buffers (rows past each step's length zeroed, so windows are unconditional).
// Per step every warp first issues the loads of v_{i-1} for kChainTch of its tiles at
// once, then computes G_{i-1} = G_i (*)^T S_i and its dS_i partials.  dS partials are
// reduced across the warps in shared memory in fixed order (deterministic, no atomics).
template <int KF, bool VEC>
__global__ void __launch_bounds__(kChainNW * 32, 2) k_chain_bwd(const ChainArgs a) {
  extern __shared__ float2 smem2[];
  constexpr int R = kChainR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Pair pr = lane_pair(a.B, lane);
  const int grows = bwd_grows(KF, a.n_max);
  float2* ring = smem2;
  float2* GA = ring + kRing * KF * kWarp;
  float2* GB = GA + (size_t)grows * kWarp;
  float2* red = GB + (size_t)grows * kWarp;  // [kChainNW][KF][32]
  pdl_wait_c();
  // backward step t handles apply i = m - t; its filter sits in ring slot t % kRing
  for (int t = 0; t < kRing - 1; ++t) {
    if (t < a.m) stage_filter<KF>(ring, t % kRing, a.filt[a.m - 1 - t], pr, lane, warp);
    cp_commit();
  }
  {
    const int nm = a.n[a.m];
    for (int r = warp; r < grows; r += kChainNW) {
      GA[r * kWarp + lane] = r < nm ? ld_rowmajor<VEC>(a.g_out + (size_t)r * a.B, pr) : make_float2(0.f, 0.f);
      GB[r * kWarp + lane] = make_float2(0.f, 0.f);
    }
  }
  cp_wait_ring();
  __syncthreads();
  const float2* G = GA + lane;
  float2* Gn = GB + lane;
  const float2* sblk =
      reinterpret_cast<const float2*>(a.states) + (size_t)blockIdx.x * a.state_rows * kWarp + lane;
  // v_{i-1} rows of the warp's first chunk of tiles are loaded into registers one step
  // ahead (at the end of step i+1), so their latency overlaps the barrier, the dS
  // reduction and the G part of the next step.
  float2 pv[kChainTch][R];
  load_prev<R>(pv, a, sblk, pr, a.m, warp * R);
  for (int t = 0; t < a.m; ++t) {
    const int i = a.m - t;
    {
      const int tt = t + kRing - 1;
      if (tt < a.m) stage_filter<KF>(ring, tt % kRing, a.filt[a.m - 1 - tt], pr, lane, warp);
      cp_commit();
    }
    float2 f[KF], d2[KF];
    {
      const float2* F = ring + (size_t)(t % kRing) * KF * kWarp + lane;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        f[j] = F[j * kWarp];
        d2[j] = make_float2(0.f, 0.f);
      }
    }
    const int nin = a.n[i - 1];
    for (int c0 = warp * R; c0 < nin; c0 += kChainTch * kChainNW * R) {
      if (c0 != warp * R) load_prev<R>(pv, a, sblk, pr, i, c0);  // chains longer than one chunk
#pragma unroll
      for (int q = 0; q < kChainTch; ++q) {
        const int s0 = c0 + q * kChainNW * R;
        if (s0 >= nin) break;
        float2 gw[R + KF - 1];
#pragma unroll
        for (int u = 0; u < R + KF - 1; ++u) gw[u] = G[(s0 + u) * kWarp];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < KF; ++j) acc = ffma2(gw[r + j], f[j], acc);
          const int s = s0 + r;
          if (i > 1)
            Gn[s * kWarp] = s < nin ? acc : make_float2(0.f, 0.f);
          else if (s < nin)
            st_strided(a.dbase_p, a.dbase_sr, a.dbase_sb, pr, s, acc);
        }
#pragma unroll
        for (int j = 0; j < KF; ++j) {
          float2 acc = d2[j];
#pragma unroll
          for (int r = 0; r < R; ++r) acc = ffma2(gw[r + j], pv[q][r], acc);
          d2[j] = acc;
        }
      }
    }
    if (i > 1)  // rows past the padded tiles that the next step's windows can reach
      for (int r = round_up(nin, R) + warp; r < nin + R + KF - 1; r += kChainNW) Gn[r * kWarp] = make_float2(0.f, 0.f);
    float2* rd = red + lane;
#pragma unroll
    for (int j = 0; j < KF; ++j) rd[(warp * KF + j) * kWarp] = d2[j];
    if (i > 1) load_prev<R>(pv, a, sblk, pr, i - 1, warp * R);
    cp_wait_ring();
    __syncthreads();
    for (int j = warp; j < KF; j += kChainNW) {
      float2 acc = rd[j * kWarp];
#pragma unroll
      for (int w = 1; w < kChainNW; ++w) {
        const float2 v = rd[(w * KF + j) * kWarp];
        acc.x += v.x;
        acc.y += v.y;
      }
      st_strided(a.dfilt_p[i - 1], a.dfilt_sr[i - 1], a.dfilt_sb[i - 1], pr, j, acc);
    }
    __syncthreads();  // red is rewritten by the next step
    const float2* tmp = G;
    G = Gn;
    Gn = const_cast<float2*>(tmp);
  }
}

template <typename... KArgs>
static cudaError_t launch_chain(void (*kernel)(KArgs...), const ChainArgs& a, size_t smem, cudaStream_t st) {
  cudaError_t e = ensure_smem((const void*)kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(a.B, kChainS));
  cfg.blockDim = dim3(kChainNW * kWarp);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

static int state_rows(int n0, int kf, int m) {
  int rows = 0, n = n0;
  for (int i = 1; i < m; ++i) {
    n += kf - 1;
    rows += n;
  }
  return rows;
}

static int fill_args(ChainArgs& a, const sg_chain* c) {
  if (c->m < 1 || c->m > kChainMaxSteps || c->kf < 1 || c->kf > 16 || c->n0 < 1) return (int)cudaErrorInvalidValue;
  a.base = CRows{c->base.ptr, c->base.stride_row, c->base.stride_b};
  a.m = c->m;
  a.B = c->B;
  a.n[0] = c->n0;
  int off = 0;
  int nmax = c->n0;
  for (int i = 1; i <= c->m; ++i) {
    a.n[i] = a.n[i - 1] + c->kf - 1;
    a.filt[i - 1] = CRows{c->filters[i - 1].ptr, c->filters[i - 1].stride_row, c->filters[i - 1].stride_b};
    a.state_off[i] = off;
    if (i < c->m) off += a.n[i];
    if (a.n[i] > nmax) nmax = a.n[i];
  }
  a.state_off[0] = 0;
  a.state_rows = off;
  a.n_max = nmax;
  a.states = c->states;
  return 0;
}

#define SG_CHAIN_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

}  // namespace sg

using namespace sg;

extern "C" {

int64_t sg_chain_states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B) {
  return (int64_t)state_rows(n0, kf, m) * (int64_t)ceil_div(B, kChainS) * kChainS;
}

int32_t sg_chain_max_rows(int32_t kf) {
  if (kf < 1 || kf > 16) return 0;
  int n = 0;
  while (fwd_smem_bytes(kf, n + 1) <= kChainSmemMax && bwd_smem_bytes(kf, n + 1) <= kChainSmemMax) ++n;
  return n;
}

int sg_chain_fwd(const sg_chain* c, float* out, sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  a.out = out;
  // all filters up front if that still leaves two CTAs per SM (or the ring would not either)
  const size_t ring_smem = fwd_smem_bytes(c->kf, a.n_max);
  const size_t all_smem = fwd_smem_bytes(c->kf, a.n_max, a.m);
  SG_RETURN_IF(ring_smem > kChainSmemMax, cudaErrorNotSupported);
  a.allf = all_smem <= kChainSmemTwo || (ring_smem > kChainSmemTwo && all_smem <= kChainSmemMax);
  const size_t smem = a.allf ? all_smem : ring_smem;
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = (c->B % 2 == 0) && ((uintptr_t)out % 8 == 0);
  switch (c->kf) {
#define X(K)                                                                \
  case K:                                                                   \
    return (int)(vec ? launch_chain(k_chain_fwd<K, true>, a, smem, st)      \
                     : launch_chain(k_chain_fwd<K, false>, a, smem, st));
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
  const size_t smem = bwd_smem_bytes(c->kf, a.n_max);
  SG_RETURN_IF(smem > kChainSmemMax, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = (c->B % 2 == 0) && ((uintptr_t)grad_out % 8 == 0);
  switch (c->kf) {
#define X(K)                                                                \
  case K:                                                                   \
    return (int)(vec ? launch_chain(k_chain_bwd<K, true>, a, smem, st)      \
                     : launch_chain(k_chain_bwd<K, false>, a, smem, st));
    SG_CHAIN_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // extern "C"
