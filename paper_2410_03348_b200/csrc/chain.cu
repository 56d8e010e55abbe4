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
// Mapping (B200).  A warp owns 16 samples for the whole chain and is self-contained: its
// state lives in its own slice of shared memory, so the 14 sequential steps of a Sum-15
// chain need only __syncwarp, never a block barrier.  Lane = (row group g = lane / 8,
// sample pair c = lane % 8): the four row groups work on four output tiles of R rows at
// once, and each lane holds the sample PAIR (2c, 2c+1), so every multiply-add is one
// packed FFMA2 (fma.rn.f32x2: two IEEE fp32 FMAs, identical rounding to two FFMAs) and
// every shared-memory access is one 8-byte LDS.64/STS.64.  Shared rows are 8 pairs + 1 pad
// (72 B), which puts the four groups' tiles (R = 8 rows apart) on alternating bank halves:
// a warp-wide LDS.64 costs the minimum two wavefronts.  Intermediate states go to HBM in a
// warp-blocked layout ([warp][row][16 samples]: one 64-byte segment per group-row).
//
// Row groups per warp (SG_CHAIN_GROUPS = 4 / 8 / 16, this file is compiled once per value,
// chain_api.cu picks one per launch from B): a warp owns 2 * 32 / G samples and each lane
// R = 32 / G rows of a 32-row round.  G = 4 gives the fewest window loads per FFMA2 and is
// best when the batch fills the GPU (B >= ~12k: 1024+ warps); smaller batches take more
// groups — fewer samples per warp, more warps, a shorter per-warp dependent chain (the
// kernels are latency-bound: at B = 2048 and G = 4 there are only 128 warps).
#include "common.cuh"

#ifndef SG_CHAIN_GROUPS
#define SG_CHAIN_GROUPS 4
#endif
#define SG_CH_CAT2(a, b) a##b
#define SG_CH_CAT(a, b) SG_CH_CAT2(a, b)
#define SG_CHAIN_NS SG_CH_CAT(chain_g, SG_CHAIN_GROUPS)

namespace sg {
namespace SG_CHAIN_NS {

constexpr int kChainMaxSteps = 32;
constexpr int kCG = SG_CHAIN_GROUPS;  // row groups per warp
constexpr int kCR = 32 / kCG;         // rows per group tile
constexpr int kPairs = 32 / kCG;      // sample pairs per group (lanes per group)
constexpr int kCWS = 2 * kPairs;      // samples per warp
constexpr int kCP = kPairs + 1;       // float2 per shared row (+1 pad: groups land on distinct bank sets)
constexpr int kRing = 4;     // cp.async filter ring depth (when not all filters are staged)
constexpr size_t kChainSmemMax = 227 * 1024;
constexpr size_t kSmSmem = 228 * 1024;  // per-SM shared memory (CTA reservation included)

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
  int state_off[kChainMaxSteps + 1];  // row offset of v_i inside a warp's state block (i = 1..m-1)
  int state_rows;                  // rows of one warp's state block
  int allf;                        // all m filters staged in shared memory up front
  int m;
  int n_max;
  int64_t B;
  float* states;       // [ceil(B/16)][state_rows][16] clamped intermediate states
  float* out;          // [n[m]][B]
  double* rowsum;      // forward, optional: [B] sum over the output rows (fp64)
  const float* g_out;  // backward: [n[m]][B]
  // backward with the fused loss (g_out == nullptr): the upstream gradient of
  // loss_nll(v_m, targets) (learn.py:92-119) is generated in place from per-sample scalars
  const double* nll_pt;        // [B] picked probabilities p[t_b][b] (sg_nll_fwd_rowsum's side output)
  const int64_t* nll_t;        // targets [B] (-1 = no mass)
  const double* nll_rowsum;    // [B] sums of v_m rows (the forward's side output)
  const double* nll_gloss;     // scalar upstream gradient of the loss
  float* dbase_p;      // backward: grad of v_0 (strided like base)
  int64_t dbase_sr, dbase_sb;
};

__device__ __forceinline__ void pdl_wait_c() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
// 8-byte cp.async with zero fill: src_bytes = 0 writes zeros without reading
__device__ __forceinline__ void cp_async8z(float2* dst, const void* src, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4z(float* dst, const float* src, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(src), "r"(src_bytes) : "memory");
}
// bulk prefetch of a contiguous global range into L2 (no registers, no shared memory)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// per-lane L1 prefetch of a contiguous range (lines lane, lane + 32, ...): the backward's
// next-step state block lands in L1 (free: the chain kernels leave most of it to L1),
// so the v_{i-1} row loads of a round hit L1 instead of waiting on L2 under load
__device__ __forceinline__ void prefetch_l1_range(const void* p, unsigned bytes, int lane) {
  const char* c = reinterpret_cast<const char*>(p);
  for (unsigned o = (unsigned)lane * 128u; o < bytes; o += 32u * 128u)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c + o));
}
#ifndef SG_CHAIN_L1PF
#define SG_CHAIN_L1PF 1
#endif
#ifndef SG_CHAIN_SATFMA
#define SG_CHAIN_SATFMA 1
#endif
// last tap of a forward output as two scalar fma.rn.sat (round, then clamp to [0, 1];
// NaN -> +0 like clamp01): bit-identical to ffma2 followed by clamp01x2, 2 instructions
// instead of 5 (FFMA2 + four FMNMX)
__device__ __forceinline__ float2 ffma2_sat(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.x) : "f"(a.x), "f"(b.x), "f"(c.x));
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d.y) : "f"(a.y), "f"(b.y), "f"(c.y));
  return d;
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_ring() { asm volatile("cp.async.wait_group %0;" ::"n"(kRing - 2) : "memory"); }

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 clamp01x2(float2 v) { return make_float2(clamp01(v.x), clamp01(v.y)); }
__device__ __forceinline__ float2 zero2() { return make_float2(0.f, 0.f); }

// What a lane owns: row group g, pair c = samples (b0, b0 + 1) of warp `wid`.  Loads use
// clamped sample indices, stores are predicated by nv (valid samples of the pair).
struct Lane {
  int g, c;
  int64_t wid, b0, ba, bb;
  int nv;
};

__device__ __forceinline__ Lane lane_of(int64_t B) {
  Lane L;
  const int lane = threadIdx.x & 31;
  L.g = lane / kPairs;
  L.c = lane % kPairs;
  L.wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  L.b0 = L.wid * kCWS + 2 * L.c;
  const int64_t left = B - L.b0;
  L.nv = left <= 0 ? 0 : (left >= 2 ? 2 : 1);
  L.ba = L.b0 < B ? L.b0 : B - 1;
  L.bb = L.b0 + 1 < B ? L.b0 + 1 : B - 1;
  return L;
}

__device__ __forceinline__ float2 ld_strided(const CRows& S, const Lane& L, int64_t row) {
  return make_float2(__ldg(S.p + L.ba * S.sb + row * S.sr), __ldg(S.p + L.bb * S.sb + row * S.sr));
}

__device__ __forceinline__ void st_strided(float* base, int64_t sr, int64_t sb, const Lane& L, int64_t row, float2 v) {
  if (L.nv > 0) base[L.b0 * sb + row * sr] = v.x;
  if (L.nv > 1) base[(L.b0 + 1) * sb + row * sr] = v.y;
}

// [rows][B] row-major (out, g_out): 8-byte vector access when B is even (then a pair is
// either fully valid or fully past the end).
template <bool VEC>
__device__ __forceinline__ float2 ld_rowmajor(const float* q, const Lane& L) {  // q = row start
  if constexpr (VEC) {
    return L.nv == 2 ? __ldg(reinterpret_cast<const float2*>(q + L.b0)) : zero2();
  } else {
    return make_float2(__ldg(q + L.ba), __ldg(q + L.bb));
  }
}

template <bool VEC>
__device__ __forceinline__ void st_rowmajor(float* q, const Lane& L, float2 v) {
  if constexpr (VEC) {
    if (L.nv == 2) *reinterpret_cast<float2*>(q + L.b0) = v;
  } else {
    if (L.nv > 0) q[L.b0] = v.x;
    if (L.nv > 1) q[L.b0 + 1] = v.y;
  }
}

// Filter S (KF rows of the warp's 16 samples) -> shared slot `slot` ([KF][kCP] float2).
// Element e = lane + 32k: row e / 16, sample e % 16 (pair, half).
template <int KF>
__device__ __forceinline__ void stage_filter(float2* F, int slot, const CRows& S, const Lane& L, int64_t B) {
  const int lane = threadIdx.x & 31;
  float* d = reinterpret_cast<float*>(F + (size_t)slot * KF * kCP);
  const int64_t wb = L.wid * kCWS;
#pragma unroll
  for (int e0 = 0; e0 < KF * kCWS; e0 += 32) {
    const int e = e0 + lane;
    if (KF * kCWS % 32 == 0 || e < KF * kCWS) {
      const int j = e / kCWS, t = e % kCWS;
      int64_t b = wb + t;
      b = b < B ? b : B - 1;
      cp_async4(d + (j * kCP + (t >> 1)) * 2 + (t & 1), S.p + b * S.sb + (int64_t)j * S.sr);
    }
  }
}

// acc[r] = sum_{j ascending} w[r + KF-1-j] * f[j] (the k_conv_fwd order), computed j
// outer / r inner so the R accumulators are independent back-to-back FFMA2s.
template <int KF, int R, bool SAT = false>
__device__ __forceinline__ void conv_tile(float2 (&acc)[R], const float2 (&w)[R + KF - 1], const float2 (&f)[KF]) {
  if constexpr (SAT && KF == 1) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = ffma2_sat(w[r + KF - 1], f[0], zero2());
    return;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = __fmul2_rn(w[r + KF - 1], f[0]);  // == fma(w, f, 0)
#pragma unroll
  for (int j = 1; j < KF; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r)
      acc[r] = (SAT && j == KF - 1) ? ffma2_sat(w[r + KF - 1 - j], f[j], acc[r]) : ffma2(w[r + KF - 1 - j], f[j], acc[r]);
}

__host__ __device__ constexpr int round_up(int a, int r) { return (a + r - 1) / r * r; }

// Shared rows of one warp's slice (kCP float2 = 72 B each).  The state is updated IN
// PLACE (one buffer): rounds of kCG tiles are warp-uniform and every round loads all its
// windows before it stores (with a __syncwarp between), so no tile overwrites a row that
// another group of the same round still has to read.
constexpr int kRound = kCG * kCR;  // rows per warp round
__host__ __device__ inline int fwd_vrows(int kf, int n_max) { return (kf - 1) + round_up(n_max, kRound); }
__host__ __device__ inline int bwd_grows(int kf, int n_max) { return round_up(n_max, kRound) + kf + kCR; }
inline size_t fwd_warp_bytes(int kf, int n_max, int fslots) {
  return (size_t)(fslots * kf + fwd_vrows(kf, n_max)) * kCP * sizeof(float2);
}
inline size_t bwd_warp_bytes(int kf, int n_max) {
  return (size_t)(kRing * kf + bwd_grows(kf, n_max) + kCG * kf) * kCP * sizeof(float2);
}
// resident warps per SM for a per-warp slice (one warp per CTA; 1 KB reserved per CTA)
inline int warps_per_sm(size_t wbytes) {
  const int w = (int)(kSmSmem / (wbytes + 1024));
  return w > 32 ? 32 : w;
}

template <int KF, int R>
__device__ __forceinline__ void fwd_window(float2 (&w)[R + KF - 1], const float2* v0, int o0) {
  const float2* p = v0 + (o0 - (KF - 1)) * kCP;
#pragma unroll
  for (int u = 0; u < R + KF - 1; ++u) w[u] = p[u * kCP];
}

// One forward round for the lane's group: rows o0..o0+R-1 of v_i from its window.
template <int KF, int R, bool VEC>
__device__ __forceinline__ void fwd_round(const float2 (&w)[R + KF - 1], const float2 (&f)[KF], float2* v0,
                                          float2* gst, int o0, int nout, bool last, bool full, const ChainArgs& a,
                                          const Lane& L, double2& rsum) {
  float2 acc[R];
  conv_tile<KF, R, SG_CHAIN_SATFMA != 0>(acc, w, f);  // SAT: acc is already clamp01'ed
  __syncwarp();  // every group's window (this round's and the next's) is loaded before any store
  if (!last) {
    // one 64-bit row pointer per round: the R stores use immediate offsets; `full` (warp-
    // uniform: every row of the round is a real row) drops the per-row bounds checks
    float2* vrow = v0 + o0 * kCP;
    float2* grow = gst + (size_t)o0 * (kCWS / 2);
    if (full) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 v = SG_CHAIN_SATFMA ? acc[r] : clamp01x2(acc[r]);
        vrow[r * kCP] = v;
        grow[r * (kCWS / 2)] = v;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 v = SG_CHAIN_SATFMA ? acc[r] : clamp01x2(acc[r]);
        vrow[r * kCP] = v;  // padded rows >= nout get clamp01(0) = 0
        if (o0 + r < nout) grow[r * (kCWS / 2)] = v;
      }
    }
  } else {
    float* q = a.out + (size_t)o0 * a.B;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (o0 + r < nout) {
        const float2 v = SG_CHAIN_SATFMA ? acc[r] : clamp01x2(acc[r]);
        st_rowmajor<VEC>(q, L, v);
        rsum.x += (double)v.x;  // per-sample sum of the output row (the loss' normaliser)
        rsum.y += (double)v.y;
      }
      q += a.B;
    }
  }
}

// Forward.  Rows >= n_{i-1} of the source buffer are always exactly 0 (never written, or
// clamp01(0) from a padded tile of an earlier, shorter step), and kf-1 zero rows sit in
// front, so every window load is unconditional.
template <int KF, bool VEC>
__global__ void __launch_bounds__(32) k_chain_fwd(const ChainArgs a) {
  extern __shared__ float2 smem2[];
  constexpr int R = kCR, PAD = KF - 1;
  const Lane L = lane_of(a.B);
  const int vrows = fwd_vrows(KF, a.n_max);
  const int fslots = a.allf ? a.m : kRing;
  float2* F = smem2;
  float2* V = F + (size_t)fslots * KF * kCP;
  pdl_wait_c();
  if (a.allf) {
    for (int s = 1; s <= a.m; ++s) stage_filter<KF>(F, s - 1, a.filt[s - 1], L, a.B);
    cp_commit();
  } else {
    for (int s = 1; s < kRing; ++s) {
      if (s <= a.m) stage_filter<KF>(F, s % kRing, a.filt[s - 1], L, a.B);
      cp_commit();
    }
  }
  for (int r = L.g; r < vrows; r += kCG) {
    const int s = r - PAD;
    const bool in = s >= 0 && s < a.n[0];
    float* d = reinterpret_cast<float*>(V + r * kCP + L.c);
    const float* q = a.base.p + (int64_t)(in ? s : 0) * a.base.sr;
    cp_async4z(d, q + L.ba * a.base.sb, in ? 4 : 0);
    cp_async4z(d + 1, q + L.bb * a.base.sb, in ? 4 : 0);
  }
  cp_commit();
  cp_wait_all();
  __syncwarp();
  float2* v0 = V + PAD * kCP + L.c;  // state row 0 of this lane's pair
  float2* sblk = reinterpret_cast<float2*>(a.states) + (size_t)L.wid * a.state_rows * (kCWS / 2) + L.c;
  double2 rsum = make_double2(0.0, 0.0);
  for (int i = 1; i <= a.m; ++i) {
    if (!a.allf) {
      const int s = i + kRing - 1;
      if (s <= a.m) stage_filter<KF>(F, s % kRing, a.filt[s - 1], L, a.B);
      cp_commit();
    }
    float2 f[KF];
    {
      const float2* Fi = F + (size_t)(a.allf ? i - 1 : i % kRing) * KF * kCP + L.c;
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = Fi[j * kCP];
    }
    const int nout = a.n[i];
    const bool last = i == a.m;
    float2* gst = sblk + (size_t)a.state_off[i] * (kCWS / 2);
    // rounds in DESCENDING row order: out[o] reads v[o-KF+1 .. o], so a round only reads
    // rows that no later (lower) round has overwritten yet -- which also lets the next
    // round's windows be loaded while this round computes (two register sets)
    const int kr = round_up(nout, kRound) / kRound;
    float2 wA[R + KF - 1], wB[R + KF - 1];
    fwd_window<KF, R>(wA, v0, (kr - 1) * kRound + L.g * R);
    for (int k = kr - 1; k >= 0; k -= 2) {
      if (k >= 1) fwd_window<KF, R>(wB, v0, (k - 1) * kRound + L.g * R);
      fwd_round<KF, R, VEC>(wA, f, v0, gst, k * kRound + L.g * R, nout, last, (k + 1) * kRound <= nout, a, L,
                            rsum);
      if (k < 1) break;
      if (k >= 2) fwd_window<KF, R>(wA, v0, (k - 2) * kRound + L.g * R);
      fwd_round<KF, R, VEC>(wB, f, v0, gst, (k - 1) * kRound + L.g * R, nout, last, k * kRound <= nout, a, L,
                            rsum);
    }
    if (!a.allf) cp_wait_ring();
    __syncwarp();
  }
  if (a.rowsum != nullptr) {  // the groups' partial row sums, combined in fixed order
#pragma unroll
    for (int o = kPairs; o < 32; o <<= 1) {
      rsum.x += __shfl_xor_sync(0xffffffffu, rsum.x, o);
      rsum.y += __shfl_xor_sync(0xffffffffu, rsum.y, o);
    }
    if (L.g == 0) {
      if (L.nv > 0) a.rowsum[L.b0] = rsum.x;
      if (L.nv > 1) a.rowsum[L.b0 + 1] = rsum.y;
    }
  }
}

// v_{ii-1} rows s0 .. s0+R-1 of step ii for the lane's pair (0 past the state's end: those
// rows meet nonzero G rows in the dS sums).  FIRST: v_0 is the (strided) base operand.
template <int R, bool FIRST>
__device__ __forceinline__ void load_prev(float2 (&pv)[R], const ChainArgs& a, const float2* sblk, const Lane& L,
                                          int ii, int s0) {
  const int nin = a.n[ii - 1];
  if constexpr (!FIRST) {
    const float2* p = sblk + (size_t)(a.state_off[ii - 1] + s0) * (kCWS / 2);
    if (s0 + R <= nin) {  // all rows real: unpredicated loads at immediate offsets
#pragma unroll
      for (int r = 0; r < R; ++r) pv[r] = p[r * (kCWS / 2)];
      return;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = s0 + r < nin ? p[r * (kCWS / 2)] : zero2();
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = s0 + r < nin ? ld_strided(a.base, L, s0 + r) : zero2();
  }
}

// One backward step (apply i), in place on G.  Rounds ascend: G_{i-1}[s] reads G_i[s ..
// s+KF-1], so a round only reads rows no earlier round has overwritten, and inside a round
// every group loads its window before any group stores (__syncwarp).  Per tile: rows
// s0..s0+R-1 of G_{i-1} = G_i (*)^T S_i (j outer / rows inner for ILP; per-row order j
// ascending as in k_conv_bwd) and the tile's dS_i partials (rows ascending, KF chains).
// The v_{i-1} rows of a group's next tile are in flight (second register set) while the
// current tile computes; pvA holds the first tile on entry and the next step's first tile
// on exit.  The four groups' dS partials are summed through shared scratch in fixed order
// (deterministic, no atomics).
template <int KF, int R>
__device__ __forceinline__ void bwd_window(float2 (&gw)[R + KF - 1], const float2* G, int s0) {
  const float2* p = G + s0 * kCP;
#pragma unroll
  for (int u = 0; u < R + KF - 1; ++u) gw[u] = p[u * kCP];
}

// gw: this round's G window, loaded by the caller one round ahead (the next round's
// windows never overlap this round's stores: rounds ascend by kRound rows)
template <int KF, int R, bool FIRST>
__device__ __forceinline__ void bwd_round(float2* G, const float2 (&f)[KF], const float2 (&gw)[R + KF - 1],
                                          const float2 (&pv)[R], float2 (&d2)[KF], int s0, int nin, bool full,
                                          const ChainArgs& a, const Lane& L) {
  float2 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = __fmul2_rn(gw[r], f[0]);  // == fma(gw, f, 0)
#pragma unroll
  for (int j = 1; j < KF; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = ffma2(gw[r + j], f[j], acc[r]);
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < KF; ++j) d2[j] = ffma2(gw[r + j], pv[r], d2[j]);
  if constexpr (!FIRST) {
    __syncwarp();  // every group's window is loaded before any group stores
    if (full) {  // warp-uniform: every row of this round is a real row
#pragma unroll
      for (int r = 0; r < R; ++r) G[(s0 + r) * kCP] = acc[r];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) G[(s0 + r) * kCP] = s0 + r < nin ? acc[r] : zero2();
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (s0 + r < nin) st_strided(a.dbase_p, a.dbase_sr, a.dbase_sb, L, s0 + r, acc[r]);
  }
}

template <int KF, int R, bool FIRST>
__device__ __forceinline__ void bwd_step(float2* G, float2* scratch, const float2 (&f)[KF], float2 (&pvA)[R], int i,
                                         const ChainArgs& a, const float2* sblk, const Lane& L) {
  constexpr int STEP = kRound;
  const int nin = a.n[i - 1];
  const int kr = round_up(nin, STEP) / STEP;  // warp-uniform round count
  float2 d2[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) d2[j] = zero2();
  float2 pvB[R];
  float2 gA[R + KF - 1], gB[R + KF - 1];
  const int s0g = L.g * R;
  bwd_window<KF, R>(gA, G, s0g);
  for (int k = 0; k < kr; k += 2) {
    const int s0 = k * STEP + s0g;
    if (k + 1 < kr) {
      load_prev<R, FIRST>(pvB, a, sblk, L, i, s0 + STEP);
      bwd_window<KF, R>(gB, G, s0 + STEP);
    }
    bwd_round<KF, R, FIRST>(G, f, gA, pvA, d2, s0, nin, (k + 1) * STEP <= nin, a, L);
    if (k + 1 >= kr) break;
    if (k + 2 < kr) {
      load_prev<R, FIRST>(pvA, a, sblk, L, i, s0 + 2 * STEP);
      bwd_window<KF, R>(gA, G, s0 + 2 * STEP);
    }
    bwd_round<KF, R, FIRST>(G, f, gB, pvB, d2, s0 + STEP, nin, (k + 2) * STEP <= nin, a, L);
  }
  if constexpr (!FIRST) {
    // rows [kr*STEP, kr*STEP + KF - 1) may still hold G_i; the next step's windows reach them
    for (int r = kr * STEP + L.g; r < kr * STEP + KF - 1; r += kCG) G[r * kCP] = zero2();
    const int nn = a.n[i - 2];
    if (i - 1 > 1) {
      load_prev<R, false>(pvA, a, sblk, L, i - 1, s0g);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) pvA[r] = s0g + r < nn ? ld_strided(a.base, L, s0g + r) : zero2();
    }
  }
  // dS_i: group partials -> scratch rows g * KF + j, summed in fixed group order
#pragma unroll
  for (int j = 0; j < KF; ++j) scratch[(L.g * KF + j) * kCP] = d2[j];
  __syncwarp();
  float* da = a.dfilt_p[i - 1] + L.b0 * a.dfilt_sb[i - 1];
  const int64_t dsr = a.dfilt_sr[i - 1], dsb = a.dfilt_sb[i - 1];
#pragma unroll
  for (int j0 = 0; j0 < KF; j0 += kCG) {
    const int j = j0 + L.g;
    if (j < KF) {
      float2 v = scratch[j * kCP];
#pragma unroll
      for (int g = 1; g < kCG; ++g) v = __fadd2_rn(v, scratch[(g * KF + j) * kCP]);
      if (L.nv > 0) da[j * dsr] = v.x;
      if (L.nv > 1) da[j * dsr + dsb] = v.y;
    }
  }
}

// Backward.  The upstream gradient G of the current step lives in one shared buffer,
// updated in place step by step (rows past each step's length zeroed, so windows are
// unconditional).
template <int KF, bool VEC>
__global__ void __launch_bounds__(32) k_chain_bwd(const ChainArgs a) {
  extern __shared__ float2 smem2[];
  constexpr int R = kCR;
  const Lane L = lane_of(a.B);
  const int grows = bwd_grows(KF, a.n_max);
  float2* F = smem2;
  float2* G = F + kRing * KF * kCP;
  float2* scratch = G + (size_t)grows * kCP;  // [kCG * KF] rows
  pdl_wait_c();
  // fused loss: the per-sample scalars (target, row sum, picked probability — independent
  // loads) are requested first, so their latency overlaps the filter staging below
  int64_t tt[2] = {0, 0};
  double rsm[2] = {0.0, 0.0}, ptv[2] = {0.0, 0.0};
  if (a.g_out == nullptr) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t bb = h == 0 ? L.ba : L.bb;
      tt[h] = __ldg(a.nll_t + bb);
      rsm[h] = __ldg(a.nll_rowsum + bb);
      ptv[h] = __ldg(a.nll_pt + bb);
    }
  }
  // backward step t handles apply i = m - t; its filter sits in ring slot t % kRing
  for (int t = 0; t < kRing - 1; ++t) {
    if (t < a.m) stage_filter<KF>(F, t % kRing, a.filt[a.m - 1 - t], L, a.B);
    cp_commit();
  }
  {
    // g_out rows -> G through cp.async (all rows in flight at once), zero-filled past the
    // last row and for samples past B; joins the first ring group
    const int nm = a.n[a.m];
    if (a.g_out == nullptr) {
      // fused loss backward: d loss / d v_m[r][b] = coef_b * ([r == t_b] / den_b - p_t / den_b^2)
      // with the fp64 scalars of k_nll_bwd (damp.cu), stored as fp32 exactly as it does
      double cf[2], cm[2], inv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t t = tt[h];
        const bool bad = t < -1 || t >= (int64_t)nm;
        const double pt = ptv[h];
        const double den = rsm[h] + 1e-8;
        const double c = fmax(t >= 0 ? fmax(pt / den, 1e-12) : 0.0, 1e-12);
        cf[h] = bad ? __longlong_as_double(0x7ff8000000000000LL) : t >= 0 ? -(__ldg(a.nll_gloss) / (double)a.B) / c : 0.0;
        cm[h] = -pt / (den * den);
        inv[h] = 1.0 / den;
      }
      // every row but the target's is (float)(cf * (0.0 + cm)) = (float)(cf * cm); the
      // target row is (float)(cf * (inv + cm)) — the same two values k_nll_bwd stores
      float gb[2], gs[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool live = L.nv > h;
        gb[h] = live ? (float)(cf[h] * cm[h]) : 0.f;
        gs[h] = live ? (float)(cf[h] * (inv[h] + cm[h])) : 0.f;
      }
      for (int r = L.g; r < grows; r += kCG) {
        float2 v = zero2();
        if (r < nm) {
          v.x = r == tt[0] ? gs[0] : gb[0];
          v.y = r == tt[1] ? gs[1] : gb[1];
        }
        G[r * kCP + L.c] = v;
      }
      cp_commit();
    } else {
    for (int r = L.g; r < grows; r += kCG) {
      const float* q = a.g_out + (size_t)(r < nm ? r : 0) * a.B;
      if (VEC) {
        cp_async8z(G + r * kCP + L.c, q + L.ba, (r < nm && L.nv == 2) ? 8 : 0);
      } else {
        float* d = reinterpret_cast<float*>(G + r * kCP + L.c);
        cp_async4z(d, q + L.ba, (r < nm && L.nv > 0) ? 4 : 0);
        cp_async4z(d + 1, q + L.bb, (r < nm && L.nv > 1) ? 4 : 0);
      }
    }
    cp_commit();
    }
  }
  const float2* sblk =
      reinterpret_cast<const float2*>(a.states) + (size_t)L.wid * a.state_rows * (kCWS / 2) + L.c;
  float2 pv[R];
  if (a.m > 1)
    load_prev<R, false>(pv, a, sblk, L, a.m, L.g * R);
  else
    load_prev<R, true>(pv, a, sblk, L, a.m, L.g * R);
  if (a.m > 2 && (threadIdx.x & 31) == 0)
    prefetch_l2_bulk(sblk - L.c + (size_t)a.state_off[a.m - 2] * (kCWS / 2), a.n[a.m - 2] * kCWS * 4);
  if (SG_CHAIN_L1PF && a.m > 1)  // v_{m-1}, read by this first step, -> L1
    prefetch_l1_range(sblk - L.c + (size_t)a.state_off[a.m - 1] * (kCWS / 2), a.n[a.m - 1] * kCWS * 4,
                      threadIdx.x & 31);
  cp_wait_all();
  __syncwarp();
  for (int t = 0; t < a.m; ++t) {
    const int i = a.m - t;
    {
      const int tt = t + kRing - 1;
      if (tt < a.m) stage_filter<KF>(F, tt % kRing, a.filt[a.m - 1 - tt], L, a.B);
      cp_commit();
    }
    float2 f[KF];
    {
      const float2* Fi = F + (size_t)(t % kRing) * KF * kCP + L.c;
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = Fi[j * kCP];
    }
    if (i > 3 && (threadIdx.x & 31) == 0)  // v_{i-3} (read in step i-2) -> L2
      prefetch_l2_bulk(sblk - L.c + (size_t)a.state_off[i - 3] * (kCWS / 2), a.n[i - 3] * kCWS * 4);
    if (SG_CHAIN_L1PF && i > 2)  // v_{i-2} (read in step i-1) -> L1 one step ahead
      prefetch_l1_range(sblk - L.c + (size_t)a.state_off[i - 2] * (kCWS / 2), a.n[i - 2] * kCWS * 4,
                        threadIdx.x & 31);
    if (i > 1)
      bwd_step<KF, R, false>(G + L.c, scratch + L.c, f, pv, i, a, sblk, L);
    else
      bwd_step<KF, R, true>(G + L.c, scratch + L.c, f, pv, i, a, sblk, L);
    cp_wait_ring();
    __syncwarp();
  }
}

template <typename... KArgs>
static cudaError_t launch_chain(void (*kernel)(KArgs...), const ChainArgs& a, size_t smem, cudaStream_t st) {
  cudaError_t e = ensure_smem((const void*)kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(a.B, kCWS));
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
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

// Entry points of this variant (declared in chain_api.cu, which exports the C ABI).
int64_t states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B) {
  return (int64_t)state_rows(n0, kf, m) * (int64_t)ceil_div(B, kCWS) * kCWS;
}

int32_t max_rows(int32_t kf) {
  if (kf < 1 || kf > 16) return 0;
  int n = 0;
  while (fwd_warp_bytes(kf, n + 1, kRing) <= kChainSmemMax && bwd_warp_bytes(kf, n + 1) <= kChainSmemMax) ++n;
  return n;
}

int fwd(const sg_chain* c, float* out, double* rowsum, sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  a.out = out;
  a.rowsum = rowsum;
  // stage all filters up front unless that costs occupancy the launch could use
  const size_t ring_bytes = fwd_warp_bytes(c->kf, a.n_max, kRing);
  const size_t all_bytes = fwd_warp_bytes(c->kf, a.n_max, a.m);
  SG_RETURN_IF(ring_bytes > kChainSmemMax, cudaErrorNotSupported);
  const int need = ceil_div(ceil_div(c->B, kCWS), 148);
  const int occ_ring = warps_per_sm(ring_bytes);
  const int occ_all = all_bytes <= kChainSmemMax ? warps_per_sm(all_bytes) : 0;
  a.allf = occ_all >= (need < occ_ring ? need : occ_ring);
  const size_t smem = a.allf ? all_bytes : ring_bytes;
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

static int chain_bwd_impl(ChainArgs& a, const sg_chain* c, sg_rows grad_base, const sg_rows* grad_filters,
                          sg_stream_t stream);

int bwd(const sg_chain* c, const float* grad_out, sg_rows grad_base, const sg_rows* grad_filters,
        sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  SG_RETURN_IF(grad_out == nullptr, cudaErrorInvalidValue);
  a.g_out = grad_out;
  return chain_bwd_impl(a, c, grad_base, grad_filters, stream);
}

int bwd_nll(const sg_chain* c, const int64_t* targets, const double* rowsum, const double* picked,
            const double* grad_loss, sg_rows grad_base, const sg_rows* grad_filters, sg_stream_t stream) {
  ChainArgs a{};
  int rc = fill_args(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  SG_RETURN_IF(picked == nullptr || targets == nullptr || rowsum == nullptr || grad_loss == nullptr,
               cudaErrorInvalidValue);
  a.g_out = nullptr;
  a.nll_pt = picked;
  a.nll_t = targets;
  a.nll_rowsum = rowsum;
  a.nll_gloss = grad_loss;
  return chain_bwd_impl(a, c, grad_base, grad_filters, stream);
}

static int chain_bwd_impl(ChainArgs& a, const sg_chain* c, sg_rows grad_base, const sg_rows* grad_filters,
                          sg_stream_t stream) {
  a.dbase_p = grad_base.ptr;
  a.dbase_sr = grad_base.stride_row;
  a.dbase_sb = grad_base.stride_b;
  for (int i = 0; i < c->m; ++i) {
    a.dfilt_p[i] = grad_filters[i].ptr;
    a.dfilt_sr[i] = grad_filters[i].stride_row;
    a.dfilt_sb[i] = grad_filters[i].stride_b;
  }
  const size_t smem = bwd_warp_bytes(c->kf, a.n_max);
  SG_RETURN_IF(smem > kChainSmemMax, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = (c->B % 2 == 0) && ((uintptr_t)a.g_out % 8 == 0);
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

}  // namespace SG_CHAIN_NS
}  // namespace sg
