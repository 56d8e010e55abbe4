// DAMP (add-mult) kernels for sm_100a.
//
// K1 forward  out[o][b]  = clamp01( sum_{c in seg(o)} prod_i p_i[s_i(c)][b] )
//      reference: distribution.py:262-270 -> provenance.py:233 gather, :236 conj (T.mul),
//                 :242-253 group_disj (dense 0/1 matmul + clamp)
// K2 backward dp_k[s][b] = sum_{c: s_k(c)=s} g[T[c]][b] * prod_{j!=k} p_j[s_j(c)][b]
//      reference: tensor.py:287 (clamp bw = identity), :415 (affine bw g @ G.T),
//                 :240 (mul bw), :386-391 (select_rows bw np.add.at)
//
// Both are one "segmented sum of products" over memoised int32 records.  Operands are
// strided [rows][B] views (sg_rows): tags our kernels produce are symbol-major (B, 1) so a
// warp's 32 lanes (= 32 samples) read one coalesced 128-byte line per row; user (B, n)
// classifier blocks are read in place with strides (1, n) — no layout copies.  Records
// are warp-uniform, each segment accumulates in registers (no atomics, no shared-memory
// read-modify-write), long segments spill partial rows to scratch and are finished by a
// deterministic fix-up pass.
//
// Toeplitz fast path (T[s0][s1] == s0 + s1 — every Sum-N fold step and the sum sweep):
// the short input lives in registers and the long one streams through a register window,
// so a combination costs one FFMA and the kernels are HBM-bound.
//
// All launches use programmatic dependent launch (PDL): a kernel's CTAs are scheduled
// while the previous kernel drains and wait on `griddepcontrol.wait` before touching
// global memory, hiding the launch gap between the short per-apply kernels.
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace sg {


__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

static bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("SG_NO_PDL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------- generic segmented sum of products -------------------
struct SegsumK {
  Rows ops[SG_MAX_ARITY];
  int32_t op_off[SG_MAX_ARITY];  // row offset of operand i inside the shared tile
  int32_t op_fo[SG_MAX_ARITY];   // resident kernel: float offset of operand i inside a group tile
  int32_t op_rows[SG_MAX_ARITY];
  int32_t clamp;
  int64_t B;
  const int32_t* recs;
  const int32_t* items;
  const int32_t* blk;
  WRows out;
  float* scratch;
};

template <int NOPS, int RW, bool STAGED>
__global__ void __launch_bounds__(256) k_segsum(const SegsumK a) {
  extern __shared__ float tile[];  // [total_rows][32]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b < a.B;
  const int64_t bs = bval ? b : (a.B - 1);
  pdl_wait();

  if constexpr (STAGED) {
#pragma unroll
    for (int i = 0; i < NOPS; ++i) {
      const Rows src = a.ops[i];
      float* dst = tile + (size_t)a.op_off[i] * kWarp + lane;
      const int rows = a.op_rows[i];
      int r = warp;
      for (; r + 3 * nwarps < rows; r += 4 * nwarps) {
        float v0 = src.ld(r, bs);
        float v1 = src.ld(r + nwarps, bs);
        float v2 = src.ld(r + 2 * nwarps, bs);
        float v3 = src.ld(r + 3 * nwarps, bs);
        dst[(size_t)r * kWarp] = v0;
        dst[(size_t)(r + nwarps) * kWarp] = v1;
        dst[(size_t)(r + 2 * nwarps) * kWarp] = v2;
        dst[(size_t)(r + 3 * nwarps) * kWarp] = v3;
      }
      for (; r < rows; r += nwarps) dst[(size_t)r * kWarp] = src.ld(r, bs);
    }
    __syncthreads();
  }

  const float* opbase[NOPS];
  int64_t ostride[NOPS];
#pragma unroll
  for (int i = 0; i < NOPS; ++i) {
    if constexpr (STAGED) {
      opbase[i] = tile + (size_t)a.op_off[i] * kWarp + lane;
      ostride[i] = kWarp;
    } else {
      opbase[i] = a.ops[i].p + bs * a.ops[i].sb;
      ostride[i] = a.ops[i].sr;
    }
  }
#define SG_VAL(i, row) (STAGED ? opbase[i][(row) * kWarp] : __ldg(opbase[i] + (int64_t)(row) * ostride[i]))

  const int it0 = __ldg(a.blk + blockIdx.y);
  const int it1 = __ldg(a.blk + blockIdx.y + 1);
  for (int it = it0 + warp; it < it1; it += nwarps) {
    const int4 item = __ldg(reinterpret_cast<const int4*>(a.items) + it);
    float acc0 = 0.f, acc1 = 0.f;
    int c = item.y;
    const int32_t* rp = a.recs + (size_t)c * RW;
    for (; c + 1 < item.z; c += 2, rp += 2 * RW) {
      Rec<RW> r0 = load_rec<RW>(rp);
      Rec<RW> r1 = load_rec<RW>(rp + RW);
      float q0 = SG_VAL(0, r0.v[0]);
      float q1 = SG_VAL(0, r1.v[0]);
#pragma unroll
      for (int i = 1; i < NOPS; ++i) {
        q0 *= SG_VAL(i, r0.v[i]);
        q1 *= SG_VAL(i, r1.v[i]);
      }
      acc0 += q0;
      acc1 += q1;
    }
    if (c < item.z) {
      Rec<RW> r0 = load_rec<RW>(rp);
      float q0 = SG_VAL(0, r0.v[0]);
#pragma unroll
      for (int i = 1; i < NOPS; ++i) q0 *= SG_VAL(i, r0.v[i]);
      acc0 += q0;
    }
    const float acc = acc0 + acc1;
    if (bval) {
      if (item.w < 0)
        a.out.st(item.x, b, a.clamp ? clamp01(acc) : acc);
      else
        a.scratch[(size_t)item.w * a.B + b] = acc;
    }
  }
#undef SG_VAL
}

// Plan-resident persistent variant for small plans (north-star kernel 1/2 on the HBM-bound
// shapes: tens of symbols, a few hundred records).  The whole plan — items and records —
// is staged once per CTA into shared memory, and each persistent CTA then walks sample
// groups of 32: the operand rows of the NEXT group stream in with cp.async while the
// current group's segments are summed from shared memory (records are warp-broadcast
// reads, operands conflict-free [row][32] lane reads), and every output row leaves as one
// coalesced 128-byte store.  No dependent global load chain per item, no re-staging per
// item chunk.  Same record order and accumulator pairing as k_segsum (bit-identical).
constexpr int kResWarps = 4;

// One record of RW int32 words from shared memory (warp-broadcast vector read).
template <int RW>
__device__ __forceinline__ Rec<RW> load_rec_s(const int32_t* p) {
  Rec<RW> r;
  if constexpr (RW == 1) {
    r.v[0] = p[0];
  } else if constexpr (RW == 2) {
    const int2 t = *reinterpret_cast<const int2*>(p);
    r.v[0] = t.x; r.v[1] = t.y;
  } else {
#pragma unroll
    for (int k = 0; k < RW; k += 4) {
      const int4 t = *reinterpret_cast<const int4*>(p + k);
      r.v[k] = t.x; r.v[k + 1] = t.y; r.v[k + 2] = t.z; r.v[k + 3] = t.w;
    }
  }
  return r;
}

__device__ __forceinline__ void cp_async4_res(float* dst, const float* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_res(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src) : "memory");
}

// SM count of the current device (cached per device).
static int sm_count_cur() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

__host__ __device__ inline size_t res_plan_bytes(int n_items, int n_recs, int rw) {
  return ((size_t)n_items * 16 + (size_t)n_recs * rw * 4 + 15) / 16 * 16;
}

template <int NOPS, int RW, bool VEC, int SM>
__global__ void __launch_bounds__(kResWarps * 32) k_segsum_res(const SegsumK a, int n_items, int n_recs,
                                                               int tile_floats, int64_t n_groups) {
  // A sample group is 64 samples: lane l holds the PAIR (b0, b0 + 1), b0 = 64 g + 2 l, so
  // every product / accumulation is one packed FMUL2 / FADD2.  Operand i is staged
  //  * symbol-major (bit i of SM clear): [row][64 samples], one conflict-free LDS.64 per
  //    read; or
  //  * sample-major (bit i set; a (B, n) block such as a user softmax output or the
  //    upstream gradient of get_probs): the group's 64 contiguous sample rows copied in
  //    16-byte chunks and read with the sample stride — no transposition copy anywhere.
  extern __shared__ __align__(16) unsigned char res_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4* items = reinterpret_cast<int4*>(res_smem);
  int32_t* recs = reinterpret_cast<int32_t*>(items + n_items);
  float* tiles = reinterpret_cast<float*>(res_smem + res_plan_bytes(n_items, n_recs, RW));
  pdl_wait();
  {  // the plan, once per CTA
    for (int i = threadIdx.x; i < n_items; i += blockDim.x) cp_async16_res(items + i, a.items + 4 * (size_t)i);
    const int rn = n_recs * RW;
    for (int i = threadIdx.x; i < rn; i += blockDim.x)
      cp_async4_res(reinterpret_cast<float*>(recs + i), reinterpret_cast<const float*>(a.recs + i));
  }
  auto stage = [&](int64_t grp, float* t) {
    const int64_t first = grp * 2 * kWarp;
    const int64_t b0 = first + 2 * lane;
    const int64_t ba = b0 < a.B ? b0 : a.B - 1;
    const int64_t bb = b0 + 1 < a.B ? b0 + 1 : a.B - 1;
#pragma unroll
    for (int i = 0; i < NOPS; ++i) {
      const Rows src = a.ops[i];
      if ((SM >> i) & 1) {
        const int64_t valid = (a.B - first) < 2 * kWarp ? (a.B - first) : 2 * kWarp;  // samples in this group
        const int64_t nfl = valid * src.sb;                                            // floats to copy
        const float* q = src.p + first * src.sb;
        float* d = t + a.op_fo[i];
        const int chunks = (int)(2 * kWarp * src.sb / 4);
        for (int k = threadIdx.x; k < chunks; k += blockDim.x) {
          const int64_t f0 = 4 * (int64_t)k;
          if (f0 < nfl && f0 + 4 > nfl) continue;    // straddles the end: element-wise below
          const int bytes = f0 + 4 <= nfl ? 16 : 0;  // past the last sample: zero fill
          const unsigned sa = (unsigned)__cvta_generic_to_shared(d + f0);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(bytes ? q + f0 : src.p),
                       "r"(bytes) : "memory");
        }
        if (nfl % 4) {  // a straddling tail chunk: element-wise
          for (int64_t f = nfl & ~3ll; f < nfl; ++f)
            if (threadIdx.x == 0) cp_async4_res(d + f, q + f);
        }
      } else {
        float* d = t + a.op_fo[i] + 2 * lane;
        const float* qa = src.p + ba * src.sb;
        const float* qb = src.p + bb * src.sb;
        for (int r = warp; r < a.op_rows[i]; r += kResWarps) {
          cp_async4_res(d + (size_t)r * 2 * kWarp, qa + (int64_t)r * src.sr);
          cp_async4_res(d + (size_t)r * 2 * kWarp + 1, qb + (int64_t)r * src.sr);
        }
      }
    }
  };
  // operand i, row r, for the lane's pair
  auto opv = [&](const float* t, int i, int r) -> float2 {
    if ((SM >> i) & 1) {
      const int64_t sb = a.ops[i].sb;
      const float* q = t + a.op_fo[i] + (int64_t)(2 * lane) * sb + r;
      return make_float2(q[0], q[sb]);
    }
    return *reinterpret_cast<const float2*>(t + a.op_fo[i] + (size_t)r * 2 * kWarp + 2 * lane);
  };
  int64_t grp = blockIdx.x;
  if (grp < n_groups) stage(grp, tiles);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int it = 0; grp < n_groups; ++it, grp += gridDim.x) {
    const int64_t nxt = grp + gridDim.x;
    if (nxt < n_groups) stage(nxt, tiles + (size_t)((it + 1) & 1) * tile_floats);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // the plan + this group's operands landed
    __syncthreads();
    const float* t = tiles + (size_t)(it & 1) * tile_floats;
    const int64_t b0 = grp * 2 * kWarp + 2 * lane;
    const int nv = b0 >= a.B ? 0 : (b0 + 1 < a.B ? 2 : 1);
    for (int itm = warp; itm < n_items; itm += kResWarps) {
      const int4 item = items[itm];
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
      int c = item.y;
      for (; c + 1 < item.z; c += 2) {
        const Rec<RW> r0 = load_rec_s<RW>(recs + (size_t)c * RW);
        const Rec<RW> r1 = load_rec_s<RW>(recs + (size_t)(c + 1) * RW);
        float2 q0 = opv(t, 0, r0.v[0]);
        float2 q1 = opv(t, 0, r1.v[0]);
#pragma unroll
        for (int i = 1; i < NOPS; ++i) {
          q0 = __fmul2_rn(q0, opv(t, i, r0.v[i]));
          q1 = __fmul2_rn(q1, opv(t, i, r1.v[i]));
        }
        acc0 = __fadd2_rn(acc0, q0);
        acc1 = __fadd2_rn(acc1, q1);
      }
      if (c < item.z) {
        const Rec<RW> r0 = load_rec_s<RW>(recs + (size_t)c * RW);
        float2 q0 = opv(t, 0, r0.v[0]);
#pragma unroll
        for (int i = 1; i < NOPS; ++i) q0 = __fmul2_rn(q0, opv(t, i, r0.v[i]));
        acc0 = __fadd2_rn(acc0, q0);
      }
      float2 acc = __fadd2_rn(acc0, acc1);
      if (item.w < 0) {
        if (a.clamp) acc = make_float2(clamp01(acc.x), clamp01(acc.y));
        float* o = a.out.p + (int64_t)item.x * a.out.sr;
        if (VEC) {
          if (nv == 2) *reinterpret_cast<float2*>(o + b0) = acc;
        } else {
          if (nv > 0) o[b0 * a.out.sb] = acc.x;
          if (nv > 1) o[(b0 + 1) * a.out.sb] = acc.y;
        }
      } else {
        float* o = a.scratch + (size_t)item.w * a.B;
        if (nv > 0) o[b0] = acc.x;
        if (nv > 1) o[b0 + 1] = acc.y;
      }
    }
    __syncthreads();  // this group's tile is restaged two groups later
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Deterministic finish of segments spread over several items (pieces summed in order).
__global__ void k_segsum_fixup(const int32_t* __restrict__ split, int n_split, const float* __restrict__ scratch,
                               int64_t B, int clamp, WRows out) {
  pdl_wait();
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  for (int s = blockIdx.y; s < n_split; s += gridDim.y) {
    const int seg = __ldg(split + 3 * s), p0 = __ldg(split + 3 * s + 1), p1 = __ldg(split + 3 * s + 2);
    float acc = 0.f;
    for (int q = p0; q < p1; ++q) acc += scratch[(size_t)q * B + b];
    out.st(seg, b, clamp ? clamp01(acc) : acc);
  }
}

template <int NOPS, int RW, bool STAGED>
static int launch_segsum_t(const SegsumK& k, int n_blocks, size_t smem, cudaStream_t st) {
  dim3 grid(ceil_div(k.B, kWarp), n_blocks);
  if (STAGED) {
    cudaError_t e = ensure_smem((const void*)k_segsum<NOPS, RW, STAGED>, smem);
    if (e != cudaSuccess) return (int)e;
  }
  cudaError_t e = launch(k_segsum<NOPS, RW, STAGED>, grid, dim3(256), STAGED ? smem : 0, st, k);
  return (int)e;
}

// Operand i is staged sample-major when it is a (B, n) row per sample (stride_row 1),
// 16-byte aligned, without a huge padding stride, and wide enough (n >= 16) that a
// per-element gather would touch a new line for nearly every sample (narrow blocks such as
// a 10-digit softmax gather better per element: their lines are reused across rows).  The
// sample stride must be odd: lane l then reads at 2 l * stride, 16 distinct banks (2-way).
static bool sample_major_ok(const Rows& r, int rows, int64_t B) {
  return B > 1 && r.sr == 1 && r.sb >= rows && rows >= 16 && (r.sb & 1) && r.sb <= 2 * (int64_t)rows + 8 &&
         ((uintptr_t)r.p % 16) == 0;
}

template <int NOPS, int RW, int SM>
static int launch_segsum_res_sm(SegsumK k, int n_items, int n_recs, cudaStream_t st) {
  int fo = 0;
  for (int i = 0; i < NOPS; ++i) {
    k.op_fo[i] = fo;
    fo += ((SM >> i) & 1) ? (int)(2 * kWarp * k.ops[i].sb) : k.op_rows[i] * 2 * kWarp;
    fo = (fo + 3) & ~3;  // 16-byte aligned operand tiles
  }
  const int tile_floats = fo;
  const size_t smem = res_plan_bytes(n_items, n_recs, RW) + 2 * (size_t)tile_floats * sizeof(float);
  const bool vec = k.out.sb == 1 && (k.out.sr % 2 == 0) && ((uintptr_t)k.out.p % 8 == 0);
  auto kern = vec ? k_segsum_res<NOPS, RW, true, SM> : k_segsum_res<NOPS, RW, false, SM>;
  cudaError_t e = ensure_smem((const void*)kern, smem);
  if (e != cudaSuccess) return (int)e;
  const int64_t groups = ceil_div(k.B, 2 * kWarp);
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  if (per_sm > 16) per_sm = 16;
  int64_t grid = (int64_t)sm_count_cur() * per_sm;
  if (grid > groups) grid = groups;
  return (int)launch(kern, dim3((unsigned)grid), dim3(kResWarps * kWarp), smem, st, k, n_items, n_recs, tile_floats,
                     groups);
}

template <int NOPS, int RW>
static int launch_segsum_res(const SegsumK& k, int n_items, int n_recs, cudaStream_t st) {
  int sm = 0;
  for (int i = 0; i < NOPS; ++i)
    if (sample_major_ok(k.ops[i], k.op_rows[i], k.B)) sm |= 1 << i;
  switch (sm) {
    case 0: return launch_segsum_res_sm<NOPS, RW, 0>(k, n_items, n_recs, st);
    case 1: return launch_segsum_res_sm<NOPS, RW, 1>(k, n_items, n_recs, st);
    case 2: if constexpr (NOPS >= 2) return launch_segsum_res_sm<NOPS, RW, 2>(k, n_items, n_recs, st); break;
    case 3: if constexpr (NOPS >= 2) return launch_segsum_res_sm<NOPS, RW, 3>(k, n_items, n_recs, st); break;
    default:
      if constexpr (NOPS >= 3) {
        switch (sm) {
          case 4: return launch_segsum_res_sm<NOPS, RW, 4>(k, n_items, n_recs, st);
          case 5: return launch_segsum_res_sm<NOPS, RW, 5>(k, n_items, n_recs, st);
          case 6: return launch_segsum_res_sm<NOPS, RW, 6>(k, n_items, n_recs, st);
          case 7: return launch_segsum_res_sm<NOPS, RW, 7>(k, n_items, n_recs, st);
        }
      }
  }
  return launch_segsum_res_sm<NOPS, RW, 0>(k, n_items, n_recs, st);
}

template <int NOPS, int RW>
static int launch_segsum_s(const SegsumK& k, bool staged, int n_blocks, size_t smem, cudaStream_t st) {
  return staged ? launch_segsum_t<NOPS, RW, true>(k, n_blocks, smem, st)
                : launch_segsum_t<NOPS, RW, false>(k, n_blocks, smem, st);
}

static constexpr size_t kMaxStageBytes = 200 * 1024;

// SG_SEGSUM_RESIDENT=0 forces the item-chunked kernel (A/B runs)
static bool res_enabled() {
  static const bool on = [] {
    const char* e = getenv("SG_SEGSUM_RESIDENT");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int run_segsum(const sg_segsum* p, const sg_rows* ops, const int32_t* op_rows, int n_ops, int64_t B, int clamp,
                      sg_rows out, float* scratch, cudaStream_t st) {
  SG_RETURN_IF(n_ops < 1 || n_ops > SG_MAX_ARITY, cudaErrorInvalidValue);
  SG_RETURN_IF(p->rec_words < n_ops, cudaErrorInvalidValue);
  if (B <= 0 || p->n_seg <= 0) return 0;
  SegsumK k{};
  int total = 0;
  for (int i = 0; i < n_ops; ++i) {
    k.ops[i] = rows_of(ops[i]);
    k.op_rows[i] = op_rows[i];
    k.op_off[i] = total;
    total += op_rows[i];
  }
  k.clamp = clamp;
  k.B = B;
  k.recs = p->recs;
  k.items = p->items;
  k.blk = p->blk;
  k.out = wrows_of(out);
  k.scratch = scratch;
  const size_t smem = (size_t)total * kWarp * sizeof(float);
  const bool staged = p->staged && smem <= kMaxStageBytes;
  int rc = 0;
  // small plan, many sample groups: the plan-resident persistent kernel
  size_t res_tiles = 0;  // two group tiles, each operand in its staging layout (bounded by 2x)
  for (int i = 0; i < n_ops; ++i)
    res_tiles += 2 * (size_t)2 * kWarp * sizeof(float) *
                 (sample_major_ok(k.ops[i], op_rows[i], B) ? (size_t)k.ops[i].sb : (size_t)op_rows[i]);
  const size_t res_smem = res_plan_bytes(p->n_items, p->n_recs, p->rec_words) + res_tiles;
  const bool resident = res_enabled() && p->n_items > 0 && n_ops <= 3 && res_smem <= 64 * 1024 &&
                        ceil_div(B, 2 * kWarp) >= 2 * sm_count_cur();
  if (resident) {
    const int rw = p->rec_words, ni = p->n_items, nr = p->n_recs;
    switch (n_ops) {
      case 1: rc = rw == 1 ? launch_segsum_res<1, 1>(k, ni, nr, st) : launch_segsum_res<1, 2>(k, ni, nr, st); break;
      case 2: rc = launch_segsum_res<2, 2>(k, ni, nr, st); break;
      default: rc = launch_segsum_res<3, 4>(k, ni, nr, st); break;
    }
    if (rc) return rc;
  } else if (p->n_items > 0) {
    const int rw = p->rec_words;
    switch (n_ops) {
      case 1: rc = rw == 1 ? launch_segsum_s<1, 1>(k, staged, p->n_blocks, smem, st)
                           : launch_segsum_s<1, 2>(k, staged, p->n_blocks, smem, st); break;
      case 2: rc = launch_segsum_s<2, 2>(k, staged, p->n_blocks, smem, st); break;
      case 3: rc = launch_segsum_s<3, 4>(k, staged, p->n_blocks, smem, st); break;
      case 4: rc = launch_segsum_s<4, 4>(k, staged, p->n_blocks, smem, st); break;
      case 5: rc = launch_segsum_s<5, 8>(k, staged, p->n_blocks, smem, st); break;
      case 6: rc = launch_segsum_s<6, 8>(k, staged, p->n_blocks, smem, st); break;
      case 7: rc = launch_segsum_s<7, 8>(k, staged, p->n_blocks, smem, st); break;
      default: rc = launch_segsum_s<8, 8>(k, staged, p->n_blocks, smem, st); break;
    }
    if (rc) return rc;
  }
  if (p->n_split > 0) {
    dim3 grid(ceil_div(B, 128), p->n_split < 65535 ? p->n_split : 65535);
    cudaError_t e = launch(k_segsum_fixup, grid, dim3(128), 0, st, p->split, p->n_split, (const float*)scratch, B,
                           clamp, wrows_of(out));
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

// ------------------------------- Toeplitz fast path -----------------------------------
// out[o][b] = clamp01( sum_{j<KF} L[o-j][b] * S[j][b] ),  o in [0, nL + KF - 1)
// Warp = (32 samples, tile of R outputs); the grid is 1-D over (sample group, tile) pairs
// so the launch is a single full wave (no wave quantisation at B = 16384).  S lives in KF
// registers, L in a register window of R + KF - 1 values: R * KF FFMA per R + 2 KF - 1
// coalesced loads, every load issued before the first FFMA (memory-level parallelism).
template <int KF, int R>
__global__ void __launch_bounds__(128, 8) k_conv_fwd(const Rows L, int nL, const Rows S, float* __restrict__ out,
                                                     int n_out, int64_t B, int n_tiles, int n_pairs) {
  const int lane = threadIdx.x & 31;
  const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  pdl_wait();
  if (pair >= n_pairs) return;
  const int grp = pair / n_tiles, t = pair - grp * n_tiles;
  const int64_t b = (int64_t)grp * kWarp + lane;
  if (b >= B) return;
  constexpr int WN = R + KF - 1;
  const int o0 = t * R;
  float f[KF];
  {
    const float* q = S.p + b * S.sb;
#pragma unroll
    for (int j = 0; j < KF; ++j, q += S.sr) f[j] = __ldg(q);
  }
  float w[WN];
  {
    const int s_first = o0 - (KF - 1);
    const float* q = L.p + b * L.sb + (int64_t)s_first * L.sr;
#pragma unroll
    for (int i = 0; i < WN; ++i, q += L.sr) {
      const int s = s_first + i;
      w[i] = (s >= 0 && s < nL) ? __ldg(q) : 0.f;
    }
  }
  pdl_trigger();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < KF; ++j) acc = fmaf(w[r + KF - 1 - j], f[j], acc);
    const int o = o0 + r;
    if (o < n_out) out[(size_t)o * B + b] = clamp01(acc);
  }
}

// dL[s][b] = sum_j g[s+j][b] * S[j][b];   dS[j][b] = sum_s g[s+j][b] * L[s][b]
// CTA = one group of 32 samples, one warp per tile of R positions of L (warps loop when
// there are more than 16 tiles).  S is staged once per CTA in shared memory; the dS
// partials of the tiles are reduced across warps in a fixed order (deterministic, no
// atomics) and written by warp 0.
template <int KF, int R>
__global__ void __launch_bounds__(128, 4) k_conv_bwd(const float* __restrict__ g, int n_out, const Rows L, int nL,
                                                     const Rows S, WRows dL, WRows dS, int64_t B, int n_tiles) {
  __shared__ float sS[KF][kWarp];
  __shared__ float red[4][KF][kWarp];
  const int lane = threadIdx.x;
  const int warp = threadIdx.y;
  const int nw = blockDim.y;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < B;
  const int64_t b = bval ? b0 : B - 1;
  constexpr int WN = R + KF - 1;
  pdl_wait();
  for (int j = warp; j < KF; j += nw) sS[j][lane] = S.ld(j, b);
  __syncthreads();
  float d2[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) d2[j] = 0.f;
  for (int t = warp; t < n_tiles; t += nw) {
    const int s0 = t * R;
    float gw[WN];
    {
      const float* q = g + (size_t)s0 * B + b;
#pragma unroll
      for (int i = 0; i < WN; ++i, q += B) gw[i] = (s0 + i < n_out) ? __ldg(q) : 0.f;
    }
    {  // dS partials first: live = window + L tile + accumulators
      float pv[R];
      const float* q = L.p + b * L.sb + (int64_t)s0 * L.sr;
#pragma unroll
      for (int r = 0; r < R; ++r, q += L.sr) pv[r] = (s0 + r < nL) ? __ldg(q) : 0.f;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        float acc = d2[j];
#pragma unroll
        for (int r = 0; r < R; ++r) acc = fmaf(gw[r + j], pv[r], acc);
        d2[j] = acc;
      }
    }
    {  // then dL: live = window + filter (re-read from shared memory)
      float f[KF];
#pragma unroll
      for (int j = 0; j < KF; ++j) f[j] = sS[j][lane];
      float* q = dL.p + b * dL.sb + (int64_t)s0 * dL.sr;
#pragma unroll
      for (int r = 0; r < R; ++r, q += dL.sr) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < KF; ++j) acc = fmaf(gw[r + j], f[j], acc);
        if (bval && s0 + r < nL) *q = acc;
      }
    }
  }
  pdl_trigger();
#pragma unroll
  for (int j = 0; j < KF; ++j) red[warp][j][lane] = d2[j];
  __syncthreads();
  for (int j = warp; j < KF; j += nw) {
    float acc = red[0][j][lane];
    for (int w = 1; w < nw; ++w) acc += red[w][j][lane];
    if (bval) dS.st(j, b, acc);
  }
}

template <int KF>
static int conv_fwd_t(const Rows& L, int nL, const Rows& S, float* out, int n_out, int64_t B, cudaStream_t st) {
  constexpr int R = 16;
  const int n_tiles = ceil_div(n_out, R);
  const int n_pairs = ceil_div(B, kWarp) * n_tiles;
  return (int)launch(k_conv_fwd<KF, R>, dim3(ceil_div(n_pairs, 4)), dim3(128), 0, st, L, nL, S, out, n_out, B,
                     n_tiles, n_pairs);
}

template <int KF, int R>
static int conv_bwd_r(const float* g, int n_out, const Rows& L, int nL, const Rows& S, const WRows& dL,
                      const WRows& dS, int64_t B, cudaStream_t st) {
  const int n_tiles = ceil_div(nL, R);
  const int nw = n_tiles < 4 ? n_tiles : 4;
  return (int)launch(k_conv_bwd<KF, R>, dim3(ceil_div(B, kWarp)), dim3(kWarp, nw), 0, st, g, n_out, L, nL, S, dL, dS,
                     B, n_tiles);
}

// Tile width by the length of L: narrow tiles keep short rows from wasting lanes of work,
// 32-wide tiles keep a 512-group batch in one wave of 4-warp CTAs for long rows.
template <int KF>
static int conv_bwd_t(const float* g, int n_out, const Rows& L, int nL, const Rows& S, const WRows& dL,
                      const WRows& dS, int64_t B, cudaStream_t st) {
  if (nL <= 16) return conv_bwd_r<KF, 8>(g, n_out, L, nL, S, dL, dS, B, st);
  if (nL <= 64) return conv_bwd_r<KF, 16>(g, n_out, L, nL, S, dL, dS, B, st);
  return conv_bwd_r<KF, 32>(g, n_out, L, nL, S, dL, dS, B, st);
}

#define SG_CONV_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

// ------------------------------- staged short-filter Toeplitz ------------------------
// The same applies as k_conv_fwd / k_conv_bwd (identical forward FMA order), for CTAs of
// 32 samples x 4 warps that first stage every operand row of their samples in shared
// memory ([rows][33]): a user (B, n) block read in place is one CONTIGUOUS span per 32
// samples (32 n floats), so it is loaded with linear, fully coalesced accesses and
// transposed on the way in — instead of every warp-wide row load touching n lines (the
// strided in-place read that made the unstaged kernels L1-wavefront bound).  Gradients are
// staged the same way on the way out, and the upstream gradient is read in place in either
// layout (no transpose copy before the backward).  Lane = sample; warps split the output
// rows (tiles of 8 rows from one register window) and the filter-gradient rows.
constexpr int kCsRows = 8;     // rows per warp tile
constexpr int kCsPitch = 33;   // shared row pitch (floats): conflict-free transposed stores
__device__ __forceinline__ int cs_div(int a, int b) { return (a + b - 1) / b; }

// rows [0, n) of X for samples b0 .. b0 + 31 -> sm[r * kCsPitch + s] (0 past B).  128
// threads: a sample-major (user (B, n)) block is read as 4 threads per sample walking
// its contiguous row (no index division, 4 loads in flight per thread); symbol-major rows
// as 32 samples x 4 rows per pass.
__device__ __forceinline__ void cs_stage(float* sm, const Rows& X, int n, int64_t B, int64_t b0) {
  const int tid = threadIdx.x;
  const int ns = (int)(B - b0 < kWarp ? B - b0 : kWarp);
  if (X.sr == 1 && X.sb != 0) {
    const int sidx = tid >> 2, k0 = tid & 3;
    const bool ok = sidx < ns;
    const float* src = X.p + (b0 + (ok ? sidx : 0)) * X.sb;
#pragma unroll 4
    for (int r = k0; r < n; r += 4) sm[r * kCsPitch + sidx] = ok ? __ldg(src + r) : 0.f;
  } else {
    const int sidx = tid & 31;
    const bool ok = sidx < ns;
    const float* src = X.p + (b0 + (ok ? sidx : 0)) * X.sb;
#pragma unroll 4
    for (int r = tid >> 5; r < n; r += 4) sm[r * kCsPitch + sidx] = ok ? __ldg(src + (int64_t)r * X.sr) : 0.f;
  }
}

// sm[r * kCsPitch + s] -> rows [0, n) of Y for samples b0 .. b0 + 31 (coalesced either way)
__device__ __forceinline__ void cs_unstage(const float* sm, const WRows& Y, int n, int64_t B, int64_t b0) {
  const int tid = threadIdx.x;
  const int ns = (int)(B - b0 < kWarp ? B - b0 : kWarp);
  if (Y.sr == 1) {
    const int sidx = tid >> 2, k0 = tid & 3;
    if (sidx < ns) {
      float* dst = Y.p + (b0 + sidx) * Y.sb;
#pragma unroll 4
      for (int r = k0; r < n; r += 4) dst[r] = sm[r * kCsPitch + sidx];
    }
  } else {
    const int sidx = tid & 31;
    if (sidx < ns) {
      float* dst = Y.p + (b0 + sidx) * Y.sb;
#pragma unroll 4
      for (int r = tid >> 5; r < n; r += 4) dst[(int64_t)r * Y.sr] = sm[r * kCsPitch + sidx];
    }
  }
}

template <int KF>
__global__ void __launch_bounds__(128) k_convs_fwd(const Rows L, int nL, const Rows S, float* __restrict__ out,
                                                   int n_out, int64_t B) {
  extern __shared__ float csm[];
  float* sS = csm;                          // [KF][33]
  float* sL = csm + KF * kCsPitch;          // [(KF - 1) zero rows + nL (+ tile slack)][33]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp;
  const int64_t b = b0 + lane;
  pdl_wait();
  cs_stage(sS, S, KF, B, b0);
  cs_stage(sL + (KF - 1) * kCsPitch, L, nL, B, b0);
  const int lrows = KF - 1 + nL;
  const int lcap = KF - 1 + cs_div(n_out, kCsRows) * kCsRows;
  for (int i = threadIdx.x; i < (KF - 1) * kCsPitch; i += blockDim.x) sL[i] = 0.f;
  for (int i = lrows * kCsPitch + threadIdx.x; i < lcap * kCsPitch; i += blockDim.x) sL[i] = 0.f;
  __syncthreads();
  pdl_trigger();
  float f[KF];
#pragma unroll
  for (int j = 0; j < KF; ++j) f[j] = sS[j * kCsPitch + lane];
  const int n_tiles = cs_div(n_out, kCsRows);
  for (int t = warp; t < n_tiles; t += 4) {
    const int o0 = t * kCsRows;
    float w[kCsRows + KF - 1];  // L rows o0 - (KF - 1) .. o0 + kCsRows - 1 (zero-padded)
#pragma unroll
    for (int u = 0; u < kCsRows + KF - 1; ++u) w[u] = sL[(o0 + u) * kCsPitch + lane];
#pragma unroll
    for (int r = 0; r < kCsRows; ++r) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < KF; ++j) acc = fmaf(w[r + KF - 1 - j], f[j], acc);  // k_conv_fwd's order
      const int o = o0 + r;
      if (o < n_out && b < B) out[(size_t)o * B + b] = clamp01(acc);
    }
  }
}

// dL[s] = sum_j g[s + j] S[j] (j ascending);  dS[j] = sum_s g[s + j] L[s] (s ascending)
template <int KF>
__global__ void __launch_bounds__(128) k_convs_bwd(const Rows g, int n_out, const Rows L, int nL, const Rows S,
                                                   WRows dL, WRows dS, int64_t B) {
  extern __shared__ float csm[];
  const int gcap = cs_div(nL, kCsRows) * kCsRows + KF;  // g rows + zero slack for the windows
  float* sS = csm;                           // [KF][33]
  float* sG = sS + KF * kCsPitch;            // [gcap][33]
  float* sL = sG + gcap * kCsPitch;          // [nL][33]
  float* sdL = sL + nL * kCsPitch;           // [nL][33]
  float* sdS = sdL + nL * kCsPitch;          // [KF][33]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp;
  pdl_wait();
  cs_stage(sS, S, KF, B, b0);
  cs_stage(sG, g, n_out, B, b0);
  cs_stage(sL, L, nL, B, b0);
  for (int i = n_out * kCsPitch + threadIdx.x; i < gcap * kCsPitch; i += blockDim.x) sG[i] = 0.f;
  __syncthreads();
  pdl_trigger();
  {
    float f[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) f[j] = sS[j * kCsPitch + lane];
    const int n_tiles = cs_div(nL, kCsRows);
    for (int t = warp; t < n_tiles; t += 4) {
      const int s0 = t * kCsRows;
      float gw[kCsRows + KF - 1];
#pragma unroll
      for (int u = 0; u < kCsRows + KF - 1; ++u) gw[u] = sG[(s0 + u) * kCsPitch + lane];
#pragma unroll
      for (int r = 0; r < kCsRows; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < KF; ++j) acc = fmaf(gw[r + j], f[j], acc);
        if (s0 + r < nL) sdL[(s0 + r) * kCsPitch + lane] = acc;
      }
    }
  }
  for (int j = warp; j < KF; j += 4) {
    float acc = 0.f;
    for (int s0 = 0; s0 < nL; ++s0) acc = fmaf(sG[(s0 + j) * kCsPitch + lane], sL[s0 * kCsPitch + lane], acc);
    sdS[j * kCsPitch + lane] = acc;
  }
  __syncthreads();
  cs_unstage(sdL, dL, nL, B, b0);
  cs_unstage(sdS, dS, KF, B, b0);
}

// ------------------------------- sample-pair short Toeplitz -------------------------
// Both lists short (the sweep's arity-2 |S| = 10, Sum-2): lane = one sample PAIR, the
// whole rows of both samples in registers, every multiply-add a packed FFMA2 (two IEEE
// FMAs, identical rounding), no shared memory and no index records.  A user (B, n)
// block read in place is one contiguous 8n-byte span per pair, loaded as n 8-byte vectors
// (half the instructions and 2x fewer L1 wavefronts per sample than per-row loads of
// strided samples); symbol-major rows load as one float2 per pair (coalesced).  The
// upstream gradient is read in either layout (no transposing copy before the backward)
// and the gradients are stored in the operands' own layouts.  Forward FMA order is
// k_conv_fwd's (bit-identical outputs).
constexpr int kCpMax = 16;  // longest operand list on this path (n_out <= 2 kCpMax - 1)

// v[r] = (X[r][b], X[r][b + 1]) for r < n, 0 past n and for a missing second sample
template <int N>
__device__ __forceinline__ void cp_load(float2 (&v)[N], const Rows& X, int n, int64_t b, bool two) {
#pragma unroll
  for (int r = 0; r < N; ++r) v[r] = make_float2(0.f, 0.f);
  const float* q = X.p + b * X.sb;
  if (X.sr == 1 && X.sb == n && two && (n & 1) == 0 && ((uintptr_t)q & 7) == 0) {
    // each sample's row is n contiguous floats at an 8-byte boundary: n / 2 float2 each
    const float2* q0 = reinterpret_cast<const float2*>(q);
    const float2* q1 = reinterpret_cast<const float2*>(q + n);
#pragma unroll
    for (int u = 0; u < N / 2; ++u) {
      if (2 * u < n) {
        const float2 a0 = __ldg(q0 + u), a1 = __ldg(q1 + u);
        v[2 * u] = make_float2(a0.x, a1.x);
        v[2 * u + 1] = make_float2(a0.y, a1.y);
      }
    }
    return;
  }
  if (X.sb == 1 && two && (X.sr & 1) == 0 && ((uintptr_t)q & 7) == 0) {  // symbol-major rows: one float2 each
#pragma unroll
    for (int r = 0; r < N; ++r)
      if (r < n) v[r] = __ldg(reinterpret_cast<const float2*>(q + (int64_t)r * X.sr));
    return;
  }
#pragma unroll
  for (int r = 0; r < N; ++r)
    if (r < n) v[r] = make_float2(X.ld(r, b), two ? X.ld(r, b + 1) : 0.f);
}

// rows r < n of v -> Y[r][b], Y[r][b + 1] (the second only when `two`)
template <int N>
__device__ __forceinline__ void cp_store(const WRows& Y, int n, int64_t b, bool two, const float2 (&v)[N]) {
  float* q = Y.p + b * Y.sb;
  if (Y.sr == 1 && Y.sb == n && two && (n & 1) == 0 && ((uintptr_t)q & 7) == 0) {
    float2* q0 = reinterpret_cast<float2*>(q);
    float2* q1 = reinterpret_cast<float2*>(q + n);
#pragma unroll
    for (int u = 0; u < N / 2; ++u) {
      if (2 * u < n) {
        q0[u] = make_float2(v[2 * u].x, v[2 * u + 1].x);
        q1[u] = make_float2(v[2 * u].y, v[2 * u + 1].y);
      }
    }
    return;
  }
  if (Y.sb == 1 && two && (Y.sr & 1) == 0 && ((uintptr_t)q & 7) == 0) {
#pragma unroll
    for (int r = 0; r < N; ++r)
      if (r < n) *reinterpret_cast<float2*>(q + (int64_t)r * Y.sr) = v[r];
    return;
  }
#pragma unroll
  for (int r = 0; r < N; ++r) {
    if (r < n) {
      Y.st(r, b, v[r].x);
      if (two) Y.st(r, b + 1, v[r].y);
    }
  }
}

template <int KF>
__global__ void __launch_bounds__(128) k_convp_fwd(const Rows L, int nL, const Rows S, float* __restrict__ out,
                                                   int n_out, int64_t B) {
  const int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = 2 * pr;
  pdl_wait();
  if (b >= B) return;
  const bool two = b + 1 < B;
  float2 l[kCpMax], f[KF];
  cp_load<kCpMax>(l, L, nL, b, two);
  {
    float2 ft[KF];
    cp_load<KF>(ft, S, KF, b, two);
#pragma unroll
    for (int j = 0; j < KF; ++j) f[j] = ft[j];
  }
  pdl_trigger();
#pragma unroll
  for (int o = 0; o < kCpMax + KF - 1; ++o) {
    if (o < n_out) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < KF; ++j)  // k_conv_fwd's order: j ascending from 0
        if (o - j >= 0 && o - j < kCpMax && o - j < nL) acc = __ffma2_rn(l[o - j < kCpMax ? o - j : 0], f[j], acc);
      const float2 v = make_float2(clamp01(acc.x), clamp01(acc.y));
      if (two && ((B & 1) == 0)) {
        *reinterpret_cast<float2*>(out + (size_t)o * B + b) = v;
      } else {
        out[(size_t)o * B + b] = v.x;
        if (two) out[(size_t)o * B + b + 1] = v.y;
      }
    }
  }
}

// dL[s] = sum_j g[s + j] S[j] (j ascending);  dS[j] = sum_s g[s + j] L[s] (s ascending)
template <int KF>
__global__ void __launch_bounds__(128) k_convp_bwd(const Rows g, int n_out, const Rows L, int nL, const Rows S,
                                                   WRows dL, WRows dS, int64_t B) {
  const int64_t pr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = 2 * pr;
  pdl_wait();
  if (b >= B) return;
  const bool two = b + 1 < B;
  constexpr int NO = kCpMax + KF - 1;
  float2 gv[NO], l[kCpMax], f[KF];
  cp_load<NO>(gv, g, n_out, b, two);
  cp_load<kCpMax>(l, L, nL, b, two);
  cp_load<KF>(f, S, KF, b, two);
  pdl_trigger();
  float2 dl[kCpMax], ds[KF];
#pragma unroll
  for (int s0 = 0; s0 < kCpMax; ++s0) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < KF; ++j) acc = __ffma2_rn(gv[s0 + j], f[j], acc);
    dl[s0] = acc;
  }
#pragma unroll
  for (int j = 0; j < KF; ++j) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int s0 = 0; s0 < kCpMax; ++s0)
      if (s0 < nL) acc = __ffma2_rn(gv[s0 + j], l[s0], acc);
    ds[j] = acc;
  }
  cp_store<kCpMax>(dL, nL, b, two, dl);
  cp_store<KF>(dS, KF, b, two, ds);
}

static bool convp_fits(int kf, int nL) { return kf <= kCpMax && nL <= kCpMax; }

template <int KF>
static int convp_fwd_t(const Rows& L, int nL, const Rows& S, float* out, int n_out, int64_t B, cudaStream_t st) {
  const int64_t pairs = (B + 1) / 2;
  return (int)launch(k_convp_fwd<KF>, dim3((unsigned)ceil_div(pairs, 128)), dim3(128), 0, st, L, nL, S, out, n_out,
                     B);
}

template <int KF>
static int convp_bwd_t(const Rows& g, int n_out, const Rows& L, int nL, const Rows& S, const WRows& dL,
                       const WRows& dS, int64_t B, cudaStream_t st) {
  const int64_t pairs = (B + 1) / 2;
  return (int)launch(k_convp_bwd<KF>, dim3((unsigned)ceil_div(pairs, 128)), dim3(128), 0, st, g, n_out, L, nL, S, dL,
                     dS, B);
}

static size_t convs_fwd_smem(int kf, int n_out) {
  return (size_t)(kf + kf - 1 + ceil_div(n_out, kCsRows) * kCsRows + kCsRows) * kCsPitch * sizeof(float);
}
static size_t convs_bwd_smem(int kf, int nL) {
  return (size_t)(kf + ceil_div(nL, kCsRows) * kCsRows + kf + 2 * nL + kf) * kCsPitch * sizeof(float);
}
static bool convs_fits(int kf, int nL, int n_out) {
  return convs_fwd_smem(kf, n_out) <= 96 * 1024 && convs_bwd_smem(kf, nL) <= 96 * 1024;
}

template <int KF>
static int convs_fwd_t(const Rows& L, int nL, const Rows& S, float* out, int n_out, int64_t B, cudaStream_t st) {
  const size_t smem = convs_fwd_smem(KF, n_out);
  cudaError_t e = ensure_smem((const void*)k_convs_fwd<KF>, smem);
  if (e != cudaSuccess) return (int)e;
  return (int)launch(k_convs_fwd<KF>, dim3(ceil_div(B, kWarp)), dim3(128), smem, st, L, nL, S, out, n_out, B);
}

template <int KF>
static int convs_bwd_t(const Rows& g, int n_out, const Rows& L, int nL, const Rows& S, const WRows& dL,
                       const WRows& dS, int64_t B, cudaStream_t st) {
  const size_t smem = convs_bwd_smem(KF, nL);
  cudaError_t e = ensure_smem((const void*)k_convs_bwd<KF>, smem);
  if (e != cudaSuccess) return (int)e;
  return (int)launch(k_convs_bwd<KF>, dim3(ceil_div(B, kWarp)), dim3(128), smem, st, g, n_out, L, nL, S, dL, dS, B);
}

// ------------------------------- long Toeplitz (both operands long) ------------------
// f = sum over two long symbol lists (sweep |S| = 100, 1000): every output is a full 1-D
// convolution per sample, O(|S|) multiply-adds per output, so this is FMA-bound, not
// HBM-bound.  y[t] = sum_{u < nh} X[t + t0 - u] H[u], X rows outside [0, nx) are 0;
// forward (X = long, H = other, t0 = 0) and both gradients (X = g, H = the other input
// reversed through a negative row stride, t0 = nh - 1) are this one kernel.  Lane =
// sample; a warp owns R consecutive outputs of 32 samples and walks only the taps that
// touch X, U at a time: U filter taps and the R + U - 1 row X window sit in registers, so
// each chunk is R*U FFMA per R + 2U - 1 coalesced 128-byte row loads.  A CTA is 4 warps =
// 4 consecutive output tiles of the same 32 samples, so H and the overlapping X windows
// are L1 hits across the CTA.
// R = 64 outputs per warp once the taps are long (more FMAs per window load), else 32.
constexpr int kLcU = 16, kLcWarps = 4;

template <int R>
__global__ void __launch_bounds__(kLcWarps * 32) k_lconv(const Rows X, int nx, const Rows H, int nh, int t0,
                                                         WRows Y, int ny, int64_t B, int tblocks, int clamp) {
  constexpr int U = kLcU;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t grp = blockIdx.x / tblocks;
  const int tile = (blockIdx.x % tblocks) * kLcWarps + warp;
  const int64_t b0 = grp * kWarp + lane;
  const int64_t b = b0 < B ? b0 : B - 1;
  pdl_wait();
  const int t = tile * R;
  if (t >= ny) return;
  float acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.f;
  // taps u that reach X for some output t' in [t, t + R): x = t' + t0 - u in [0, nx)
  const int u_lo = max(0, t + t0 - nx + 1);
  const int u_hi = min(nh, t + t0 + R);
  for (int u0 = u_lo; u0 < u_hi; u0 += U) {
    float h[U];
#pragma unroll
    for (int k = 0; k < U; ++k) h[k] = u0 + k < u_hi ? H.ld(u0 + k, b) : 0.f;
    const int base = t + t0 - u0 - (U - 1);  // X row of w[0]
    float w[R + U - 1];
    if (base >= 0 && base + R + U - 2 < nx) {
#pragma unroll
      for (int k = 0; k < R + U - 1; ++k) w[k] = X.ld(base + k, b);
    } else {
#pragma unroll
      for (int k = 0; k < R + U - 1; ++k) {
        const int x = base + k;
        w[k] = (x >= 0 && x < nx) ? X.ld(x, b) : 0.f;
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fmaf(w[r + U - 1 - k], h[k], acc[r]);
  }
  if (b0 >= B) return;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (t + r < ny) Y.st(t + r, b0, clamp ? clamp01(acc[r]) : acc[r]);
}

template <int R>
static int lconv_t(const Rows& X, int nx, const Rows& H, int nh, int t0, const WRows& Y, int ny, int64_t B, int clamp,
                   cudaStream_t st) {
  const int tiles = ceil_div(ny, R);
  const int tblocks = ceil_div(tiles, kLcWarps);
  const int64_t blocks = (int64_t)ceil_div(B, kWarp) * tblocks;
  SG_RETURN_IF(blocks > 0x7fffffff, cudaErrorInvalidValue);
  return (int)launch(k_lconv<R>, dim3((unsigned)blocks), dim3(kLcWarps * kWarp), 0, st, X, nx, H, nh, t0, Y, ny, B,
                     tblocks, clamp);
}

static int lconv(const Rows& X, int nx, const Rows& H, int nh, int t0, const WRows& Y, int ny, int64_t B, int clamp,
                 cudaStream_t st) {
  return nh >= 256 ? lconv_t<64>(X, nx, H, nh, t0, Y, ny, B, clamp, st)
                   : lconv_t<32>(X, nx, H, nh, t0, Y, ny, B, clamp, st);
}

static Rows reversed(const Rows& r, int n) { return Rows{r.p + (int64_t)(n - 1) * r.sr, -r.sr, r.sb}; }

// The staged kernels are exact but measured SLOWER than the unstaged ones at the sweep's
// shapes (B=65536, arity 2, |S|=10: fwd 14.4 vs 8.2 us, bwd 20.5 vs 12.0 + 8.1 us for the
// transposing copy it removes; profiles/r02_sweep_launches.md), so they are opt-in:
// SG_CONV_STAGED=1 in the environment.
static bool conv_staged(int kf, int nL, int n_out) {
  static const bool on = [] {
    const char* e = getenv("SG_CONV_STAGED");
    return e != nullptr && e[0] == '1';
  }();
  return on && convs_fits(kf, nL, n_out);
}

static int conv_fwd(int kf, const Rows& L, int nL, const Rows& S, float* out, int n_out, int64_t B, cudaStream_t st) {
  if (convp_fits(kf, nL)) {
    switch (kf) {
#define X(K) \
  case K: return convp_fwd_t<K>(L, nL, S, out, n_out, B, st);
      SG_CONV_CASES(X)
#undef X
      default: return (int)cudaErrorInvalidValue;
    }
  }
  const bool staged = conv_staged(kf, nL, n_out);
  switch (kf) {
#define X(K) \
  case K: return staged ? convs_fwd_t<K>(L, nL, S, out, n_out, B, st) : conv_fwd_t<K>(L, nL, S, out, n_out, B, st);
    SG_CONV_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

// g: the staged kernel reads any layout; the unstaged one needs contiguous [n_out][B]
static int conv_bwd(int kf, const Rows& g, int n_out, const Rows& L, int nL, const Rows& S, const WRows& dL,
                    const WRows& dS, int64_t B, cudaStream_t st) {
  if (convp_fits(kf, nL)) {
    switch (kf) {
#define X(K) \
  case K: return convp_bwd_t<K>(g, n_out, L, nL, S, dL, dS, B, st);
      SG_CONV_CASES(X)
#undef X
      default: return (int)cudaErrorInvalidValue;
    }
  }
  if (conv_staged(kf, nL, n_out)) {
    switch (kf) {
#define X(K) \
  case K: return convs_bwd_t<K>(g, n_out, L, nL, S, dL, dS, B, st);
      SG_CONV_CASES(X)
#undef X
      default: return (int)cudaErrorInvalidValue;
    }
  }
  SG_RETURN_IF((B > 1 && g.sb != 1) || (n_out > 1 && g.sr != B), cudaErrorInvalidValue);
  switch (kf) {
#define X(K) \
  case K: return conv_bwd_t<K>(g.p, n_out, L, nL, S, dL, dS, B, st);
    SG_CONV_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

// ------------------------------- union / disjunction --------------------------------
__global__ void k_rows_add(const Rows A, const int32_t* __restrict__ ia, const Rows Bm,
                           const int32_t* __restrict__ ib, int64_t n_rows, int64_t B, int clamp,
                           float* __restrict__ out) {
  pdl_wait();
  for (int64_t r = blockIdx.y; r < n_rows; r += gridDim.y) {
    const int xa = __ldg(ia + r);
    const int xb = __ldg(ib + r);
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
      float v = 0.f;
      if (xa >= 0) v += A.ld(xa, b);
      if (xb >= 0) v += Bm.ld(xb, b);
      out[(size_t)r * B + b] = clamp ? clamp01(v) : v;
    }
  }
}

// ------------------------------- fused loss_nll -------------------------------------
// Row sums are computed in parallel over (sample tile, row chunk) — chunks are added
// when the batch alone cannot fill the GPU (HWF: B = 64, 8332 output symbols) — into
// fp64 partials [chunks][B]; a second pass finishes per sample.  Forward: per-CTA log
// terms, the last CTA to finish (ticket counter, self-resetting) sums them in CTA order.
// Backward: one pass writes every gradient row of its chunk.  Deterministic throughout.
constexpr int kNllWarps = 8;

static int nll_chunks(int64_t n, int64_t B, bool backward = false) {
  const int tiles = ceil_div(B, kWarp);
  // enough CTAs to fill the GPU; the forward also keeps few enough partials that its
  // per-sample finish (one thread per sample sums `chunks` partials) stays short at small
  // batches — the backward has no such finish, so it keeps the full 2 waves
  int want = ceil_div(2 * 148, tiles);
  if (!backward && want > 32) want = 32;
  const int max_chunks = ceil_div(n, 4 * kNllWarps);
  if (want > max_chunks) want = max_chunks;
  return want < 1 ? 1 : want;
}

__global__ void __launch_bounds__(256) k_nll_partial(const Rows p, int n, int64_t B, int rows_per,
                                                     double* __restrict__ part) {
  __shared__ double red[kNllWarps][kWarp];
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const int64_t b = b0 < B ? b0 : B - 1;
  pdl_wait();
  const int r0 = blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
  double acc0 = 0.0, acc1 = 0.0;
  int r = r0 + warp;
  for (; r + kNllWarps < r1; r += 2 * kNllWarps) {
    acc0 += (double)p.ld(r, b);
    acc1 += (double)p.ld(r + kNllWarps, b);
  }
  if (r < r1) acc0 += (double)p.ld(r, b);
  red[warp][lane] = acc0 + acc1;
  __syncthreads();
  if (warp == 0 && b0 < B) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kNllWarps; ++w) t += red[w][lane];
    part[(size_t)blockIdx.y * B + b0] = t;
  }
}

__device__ __forceinline__ double nll_rowsum(const double* __restrict__ part, int chunks, int64_t B, int64_t b) {
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(size_t)c * B + b];
  return s;
}

// Targets outside [-1, n) (the reference raises IndexError, learn.py:104-112; the host
// wrapper checks them before launch whenever it can) never index memory: the sample's log
// term and gradient become NaN, so a bad device-side target cannot pass silently.
__device__ __forceinline__ bool nll_bad_target(int64_t t, int n) { return t < -1 || t >= (int64_t)n; }

__device__ __forceinline__ double nll_picked(double s, double pt, int64_t t) {
  const double norm = pt / (s + 1e-8);
  const double fl = fmax(norm, 1e-12);
  return fmax(t >= 0 ? fl : 0.0, 1e-12);
}

// Sum of the CTA's log terms (v: this thread's term); the last CTA to finish
// (self-resetting ticket) adds the per-CTA partials in CTA order -> *loss.
__device__ __forceinline__ void nll_finish(double v, double* __restrict__ loss, double* __restrict__ blocks,
                                           unsigned* __restrict__ counter, int64_t B) {
  __shared__ double red[32];
  __shared__ bool last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nthreads = blockDim.x * blockDim.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (nthreads >> 5); ++w) t += red[w];
    blocks[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the whole last CTA adds the partials: thread i sums i, i + T, ... (fixed order), then a
  // fixed shuffle tree and warp order -> deterministic
  __threadfence();
  double t = 0.0;
  for (unsigned i = tid; i < gridDim.x; i += nthreads) t += __ldcg(blocks + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = t;
  __syncthreads();
  if (tid == 0) {
    double u = 0.0;
    for (int w = 0; w < (nthreads >> 5); ++w) u += red[w];
    *loss = -u / (double)B;
    *counter = 0u;  // self-reset for the next launch / graph replay
  }
}

// Two-pass finish (chunks > 1): per-sample sums from the chunk partials.
__global__ void __launch_bounds__(256) k_nll_fwd(const Rows p, int n, int64_t B, const int64_t* __restrict__ targets,
                                                 const double* __restrict__ part, int chunks,
                                                 double* __restrict__ rowsum, double* __restrict__ loss,
                                                 double* __restrict__ blocks, unsigned* __restrict__ counter) {
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  double v = 0.0;
  if (b0 < B) {
    const int64_t t = __ldg(targets + b0);
    const double s = nll_rowsum(part, chunks, B, b0);
    rowsum[b0] = s;
    const bool bad = nll_bad_target(t, n);
    const double pt = t >= 0 && !bad ? (double)p.ld(t, b0) : 0.0;
    v = bad ? __longlong_as_double(0x7ff8000000000000LL) : log(nll_picked(s, pt, t));
  }
  nll_finish(v, loss, blocks, counter, B);
}

// Row sums already known (the fused Sum-N chain forward writes them as a side output):
// only the picked probability and the log term per sample remain.
__global__ void __launch_bounds__(256) k_nll_fwd_given(const Rows p, int n, int64_t B,
                                                       const int64_t* __restrict__ targets,
                                                       const double* __restrict__ rowsum, double* __restrict__ loss,
                                                       double* __restrict__ blocks, unsigned* __restrict__ counter,
                                                       double* __restrict__ picked) {
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  double v = 0.0;
  if (b0 < B) {
    const int64_t t = __ldg(targets + b0);
    const bool bad = nll_bad_target(t, n);
    const double pt = t >= 0 && !bad ? (double)p.ld(t, b0) : 0.0;
    v = bad ? __longlong_as_double(0x7ff8000000000000LL) : log(nll_picked(__ldg(rowsum + b0), pt, t));
    if (picked != nullptr) picked[b0] = pt;  // p[t_b][b] for a fused backward (sg_chain_bwd_nll)
  }
  nll_finish(v, loss, blocks, counter, B);
}

// One-pass forward (chunks == 1): a CTA sums all rows of its 32 samples (warps split the
// rows, same order as k_nll_partial), then finishes their log terms.
__global__ void __launch_bounds__(256) k_nll_fwd1(const Rows p, int n, int64_t B, const int64_t* __restrict__ targets,
                                                  double* __restrict__ rowsum, double* __restrict__ loss,
                                                  double* __restrict__ blocks, unsigned* __restrict__ counter) {
  __shared__ double red[kNllWarps][kWarp];
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const int64_t b = b0 < B ? b0 : B - 1;
  pdl_wait();
  // rows warp, warp + W, ...: 8 loads in flight per thread, added in row order
  double acc0 = 0.0, acc1 = 0.0;
  int r = warp;
  for (; r + 7 * kNllWarps < n; r += 8 * kNllWarps) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = p.ld(r + k * kNllWarps, b);
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      acc0 += (double)x[k];
      acc1 += (double)x[k + 1];
    }
  }
  for (; r + kNllWarps < n; r += 2 * kNllWarps) {
    acc0 += (double)p.ld(r, b);
    acc1 += (double)p.ld(r + kNllWarps, b);
  }
  if (r < n) acc0 += (double)p.ld(r, b);
  red[warp][lane] = acc0 + acc1;
  __syncthreads();
  double v = 0.0;
  if (warp == 0 && b0 < B) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kNllWarps; ++w) s += red[w][lane];
    rowsum[b0] = s;
    const int64_t t = __ldg(targets + b0);
    const bool bad = nll_bad_target(t, n);
    const double pt = t >= 0 && !bad ? (double)p.ld(t, b0) : 0.0;
    v = bad ? __longlong_as_double(0x7ff8000000000000LL) : log(nll_picked(s, pt, t));
  }
  nll_finish(v, loss, blocks, counter, B);
}

__global__ void __launch_bounds__(256) k_nll_bwd(const Rows p, int n, int64_t B, const int64_t* __restrict__ targets,
                                                 const double* __restrict__ gloss, const double* __restrict__ rowsum,
                                                 int rows_per, WRows grad) {
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int64_t b = (int64_t)blockIdx.x * kWarp + lane;
  pdl_wait();
  if (b >= B) return;
  const int64_t t = __ldg(targets + b);
  const bool bad = nll_bad_target(t, n);
  const double s = rowsum[b];
  const double pt = t >= 0 && !bad ? (double)p.ld(t, b) : 0.0;
  const double c = nll_picked(s, pt, t);
  const double den = s + 1e-8;
  const double coef = bad ? __longlong_as_double(0x7ff8000000000000LL) : t >= 0 ? -(*gloss / (double)B) / c : 0.0;
  const double common = -pt / (den * den);
  const int r0 = blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
  for (int r = r0 + warp; r < r1; r += kNllWarps) {
    const double d = (r == t ? 1.0 / den : 0.0) + common;
    grad.st(r, b, (float)(coef * d));
  }
}

// ------------------------------- row gather / layout ---------------------------------
template <typename V>
__global__ void k_rows_gather(const V* __restrict__ src, const int32_t* __restrict__ idx, int64_t n_rows,
                              int64_t row_vecs, V* __restrict__ dst) {
  pdl_wait();
  for (int64_t r = blockIdx.y; r < n_rows; r += gridDim.y) {
    const int x = __ldg(idx + r);
    V* d = dst + (size_t)r * row_vecs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < row_vecs;
         i += (int64_t)gridDim.x * blockDim.x) {
      if (x >= 0)
        d[i] = src[(size_t)x * row_vecs + i];
      else
        d[i] = V{};
    }
  }
}

template <typename T>
__device__ __forceinline__ float to_f(T v) { return (float)v; }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v) { return (T)v; }
template <>
__device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// dst[n][B] fp32 <- src(B, n) strided (32x32 tile transpose, both sides coalesced)
template <typename T>
__global__ void k_to_symbol_major(const T* __restrict__ src, int64_t B, int64_t n, int64_t sb, int64_t sn,
                                  float* __restrict__ dst) {
  __shared__ float t[32][33];
  pdl_wait();
  const int64_t b0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t bb = b0 + i, nn = n0 + threadIdx.x;
    if (bb < B && nn < n) t[i][threadIdx.x] = to_f<T>(src[bb * sb + nn * sn]);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t nn = n0 + i, bb = b0 + threadIdx.x;
    if (bb < B && nn < n) dst[nn * B + bb] = t[threadIdx.x][i];
  }
}

template <typename T>
__global__ void k_from_symbol_major(const float* __restrict__ src, int64_t B, int64_t n, T* __restrict__ dst,
                                    int64_t sb, int64_t sn) {
  __shared__ float t[32][33];
  pdl_wait();
  const int64_t b0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t nn = n0 + i, bb = b0 + threadIdx.x;
    if (bb < B && nn < n) t[i][threadIdx.x] = src[nn * B + bb];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t bb = b0 + i, nn = n0 + threadIdx.x;
    if (bb < B && nn < n) dst[bb * sb + nn * sn] = from_f<T>(t[threadIdx.x][i]);
  }
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_version(void) { return 2; }

int sg_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

int64_t sg_launch_count(void) { return (int64_t)g_launches.load(); }

int sg_segsum_run(const sg_segsum* prob, const sg_rows* ops, const int32_t* op_rows, int32_t n_ops, int64_t B,
                  int32_t clamp01_, sg_rows out, float* scratch, sg_stream_t stream) {
  return run_segsum(prob, ops, op_rows, n_ops, B, clamp01_, out, scratch, (cudaStream_t)stream);
}

int sg_damp_apply_fwd(const sg_damp_plan* plan, const sg_rows* inputs, int64_t B, float* out, float* scratch,
                      sg_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  SG_RETURN_IF(plan->arity < 1 || plan->arity > SG_MAX_ARITY, cudaErrorInvalidValue);
  if (B <= 0 || plan->n_out <= 0) return 0;
  if (plan->conv == 3) {  // f = a + b + c: (a (*) b) (*) c, unclamped in between; scratch = a (*) b
    SG_RETURN_IF(scratch == nullptr, cudaErrorInvalidValue);
    const int n01 = plan->sizes[0] + plan->sizes[1] - 1;
    int rc = lconv(rows_of(inputs[0]), plan->sizes[0], rows_of(inputs[1]), plan->sizes[1], 0,
                   WRows{scratch, B, 1}, n01, B, 0, st);
    if (rc) return rc;
    return lconv(Rows{scratch, B, 1}, n01, rows_of(inputs[2]), plan->sizes[2], 0, WRows{out, B, 1}, plan->n_out, B, 1,
                 st);
  }
  if (plan->conv == 2) {  // long Toeplitz: out[o] = sum_j in0[o - j] in1[j]
    return lconv(rows_of(inputs[0]), plan->sizes[0], rows_of(inputs[1]), plan->sizes[1], 0,
                 WRows{out, B, 1}, plan->n_out, B, 1, st);
  }
  if (plan->conv) {
    const int sh = plan->conv_short, lo = 1 - sh;
    return conv_fwd(plan->sizes[sh], rows_of(inputs[lo]), plan->sizes[lo], rows_of(inputs[sh]), out, plan->n_out, B,
                    st);
  }
  sg_rows o{out, B, 1};
  return run_segsum(&plan->fwd, inputs, plan->sizes, plan->arity, B, 1, o, scratch, st);
}

int sg_damp_apply_bwd(const sg_damp_plan* plan, const sg_rows* inputs, sg_rows grad_rows, int64_t B,
                      const sg_rows* grad_in, float* scratch, sg_stream_t stream) {
  const Rows g = rows_of(grad_rows);
  cudaStream_t st = (cudaStream_t)stream;
  const int n = plan->arity;
  SG_RETURN_IF(n < 1 || n > SG_MAX_ARITY, cudaErrorInvalidValue);
  if (B <= 0) return 0;
  if (plan->conv == 3) {  // scratch = [t = a (*) b | dt = g corr c]; dc = g corr t, da = dt corr b, db = dt corr a
    SG_RETURN_IF(scratch == nullptr, cudaErrorInvalidValue);
    const int n0 = plan->sizes[0], n1 = plan->sizes[1], n2 = plan->sizes[2], n01 = n0 + n1 - 1;
    float* t = scratch;
    float* dt = scratch + (size_t)n01 * B;
    int rc = 0;
    if (grad_in[2].ptr != nullptr) {
      rc = lconv(rows_of(inputs[0]), n0, rows_of(inputs[1]), n1, 0, WRows{t, B, 1}, n01, B, 0, st);
      if (rc) return rc;
      rc = lconv(g, plan->n_out, reversed(Rows{t, B, 1}, n01), n01, n01 - 1, wrows_of(grad_in[2]), n2, B, 0, st);
      if (rc) return rc;
    }
    if (grad_in[0].ptr == nullptr && grad_in[1].ptr == nullptr) return 0;
    rc = lconv(g, plan->n_out, reversed(rows_of(inputs[2]), n2), n2, n2 - 1, WRows{dt, B, 1}, n01, B, 0, st);
    if (rc) return rc;
    const Rows dtr{dt, B, 1};
    if (grad_in[0].ptr != nullptr) {
      rc = lconv(dtr, n01, reversed(rows_of(inputs[1]), n1), n1, n1 - 1, wrows_of(grad_in[0]), n0, B, 0, st);
      if (rc) return rc;
    }
    if (grad_in[1].ptr != nullptr)
      rc = lconv(dtr, n01, reversed(rows_of(inputs[0]), n0), n0, n0 - 1, wrows_of(grad_in[1]), n1, B, 0, st);
    return rc;
  }
  if (plan->conv == 2) {  // d in_k[s] = sum_j g[s + j] in_other[j]: correlation = conv with the other reversed
    for (int k = 0; k < 2; ++k) {
      if (grad_in[k].ptr == nullptr) continue;
      const int o = 1 - k;
      int rc = lconv(g, plan->n_out, reversed(rows_of(inputs[o]), plan->sizes[o]), plan->sizes[o],
                     plan->sizes[o] - 1, wrows_of(grad_in[k]), plan->sizes[k], B, 0, st);
      if (rc) return rc;
    }
    return 0;
  }
  if (plan->conv) {
    const int sh = plan->conv_short, lo = 1 - sh;
    SG_RETURN_IF(grad_in[0].ptr == nullptr || grad_in[1].ptr == nullptr, cudaErrorInvalidValue);
    return conv_bwd(plan->sizes[sh], g, plan->n_out, rows_of(inputs[lo]), plan->sizes[lo], rows_of(inputs[sh]),
                    wrows_of(grad_in[lo]), wrows_of(grad_in[sh]), B, st);
  }
  for (int k = 0; k < n; ++k) {
    if (grad_in[k].ptr == nullptr) continue;
    sg_rows ops[SG_MAX_ARITY];
    int32_t rows[SG_MAX_ARITY];
    ops[0] = grad_rows;
    rows[0] = plan->n_out;
    int m = 1;
    for (int j = 0; j < n; ++j) {
      if (j == k) continue;
      ops[m] = inputs[j];
      rows[m] = plan->sizes[j];
      ++m;
    }
    int rc = run_segsum(&plan->bwd[k], ops, rows, n, B, 0, grad_in[k], scratch, st);
    if (rc) return rc;
  }
  return 0;
}

int sg_damp_rows_add(const sg_rows A, const int32_t* ia, const sg_rows Bm, const int32_t* ib, int64_t n_rows,
                     int64_t B, int32_t clamp01_, float* out, sg_stream_t stream) {
  if (n_rows <= 0 || B <= 0) return 0;
  const int threads = 256;
  int gx = ceil_div(B, threads);
  if (gx > 64) gx = 64;
  dim3 grid(gx, n_rows < 65535 ? (unsigned)n_rows : 65535u);
  return (int)launch(k_rows_add, grid, dim3(threads), 0, (cudaStream_t)stream, rows_of(A), ia, rows_of(Bm), ib,
                     n_rows, B, (int)clamp01_, out);
}

int32_t sg_damp_conv_staged(int32_t kf, int32_t n_long, int32_t n_out) {
  return (convp_fits(kf, n_long) || conv_staged(kf, n_long, n_out)) ? 1 : 0;
}

int64_t sg_nll_scratch_bytes(int64_t n, int64_t B) {
  const int chunks = nll_chunks(n, B);
  const int blocks = ceil_div(B, kWarp);
  return (int64_t)(2 + blocks + (chunks > 1 ? (int64_t)chunks * B : 0)) * (int64_t)sizeof(double);
}

// scratch layout (doubles): [0] ticket counter (zero-initialised once, self-resetting),
// [2, 2 + blocks) per-CTA log-term partials, then [chunks][B] row-sum partials (chunks > 1).
int sg_nll_fwd(sg_rows probs, int64_t n, int64_t B, const int64_t* targets, double* loss, void* scratch,
               double* rowsum, sg_stream_t stream) {
  if (B <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int chunks = nll_chunks(n, B);
  double* base = (double*)scratch;
  unsigned* counter = (unsigned*)base;
  double* blk = base + 2;
  if (chunks == 1)
    return (int)launch(k_nll_fwd1, dim3(ceil_div(B, kWarp)), dim3(kWarp, kNllWarps), 0, st, rows_of(probs), (int)n,
                       B, targets, rowsum, loss, blk, counter);
  const int rows_per = ceil_div(n, chunks);
  const int blocks = ceil_div(B, 256);
  double* part = base + 2 + ceil_div(B, kWarp);
  cudaError_t e = launch(k_nll_partial, dim3(ceil_div(B, kWarp), chunks), dim3(kWarp, kNllWarps), 0, st,
                         rows_of(probs), (int)n, B, rows_per, part);
  if (e != cudaSuccess) return (int)e;
  return (int)launch(k_nll_fwd, dim3(blocks), dim3(256), 0, st, rows_of(probs), (int)n, B, targets,
                     (const double*)part, chunks,
                     rowsum, loss, blk, counter);
}

int sg_nll_fwd_rowsum(sg_rows probs, int64_t n, int64_t B, const int64_t* targets, const double* rowsum,
                      double* loss, void* scratch, double* picked, sg_stream_t stream) {
  if (B <= 0) return 0;
  double* base = (double*)scratch;
  return (int)launch(k_nll_fwd_given, dim3(ceil_div(B, 256)), dim3(256), 0, (cudaStream_t)stream, rows_of(probs),
                     (int)n, B, targets, rowsum, loss, base + 2, (unsigned*)base, picked);
}

int sg_nll_bwd(sg_rows probs, int64_t n, int64_t B, const int64_t* targets, const double* grad_loss,
               const double* rowsum, sg_rows grad, sg_stream_t stream) {
  if (B <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int chunks = nll_chunks(n, B, /*backward=*/true);
  const int rows_per = ceil_div(n, chunks);
  return (int)launch(k_nll_bwd, dim3(ceil_div(B, kWarp), chunks), dim3(kWarp, kNllWarps), 0, st, rows_of(probs),
                     (int)n, B, targets, grad_loss, rowsum, rows_per, wrows_of(grad));
}

int sg_rows_gather(const void* src, const int32_t* idx, int64_t n_rows, int64_t row_bytes, void* dst,
                   sg_stream_t stream) {
  if (n_rows <= 0 || row_bytes <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const uintptr_t al = (uintptr_t)src | (uintptr_t)dst;
  dim3 grid(1, n_rows < 65535 ? (unsigned)n_rows : 65535u);
  const int threads = 256;
  cudaError_t e;
  if (row_bytes % 16 == 0 && al % 16 == 0) {
    const int64_t v = row_bytes / 16;
    grid.x = ceil_div(v, threads) < 32 ? ceil_div(v, threads) : 32;
    e = launch(k_rows_gather<uint4>, grid, dim3(threads), 0, st, (const uint4*)src, idx, n_rows, v, (uint4*)dst);
  } else if (row_bytes % 4 == 0 && al % 4 == 0) {
    const int64_t v = row_bytes / 4;
    grid.x = ceil_div(v, threads) < 32 ? ceil_div(v, threads) : 32;
    e = launch(k_rows_gather<uint32_t>, grid, dim3(threads), 0, st, (const uint32_t*)src, idx, n_rows, v,
               (uint32_t*)dst);
  } else {
    grid.x = ceil_div(row_bytes, threads) < 32 ? ceil_div(row_bytes, threads) : 32;
    e = launch(k_rows_gather<uint8_t>, grid, dim3(threads), 0, st, (const uint8_t*)src, idx, n_rows, row_bytes,
               (uint8_t*)dst);
  }
  return (int)e;
}

int sg_to_symbol_major(const void* src, int32_t src_dtype, int64_t B, int64_t n, int64_t stride_b, int64_t stride_n,
                       float* dst, sg_stream_t stream) {
  if (B <= 0 || n <= 0) return 0;
  dim3 block(32, 8), grid(ceil_div(B, 32), ceil_div(n, 32));
  cudaStream_t st = (cudaStream_t)stream;
  switch (src_dtype) {
    case 0: return (int)launch(k_to_symbol_major<float>, grid, block, 0, st, (const float*)src, B, n, stride_b,
                               stride_n, dst);
    case 1: return (int)launch(k_to_symbol_major<double>, grid, block, 0, st, (const double*)src, B, n, stride_b,
                               stride_n, dst);
    case 2: return (int)launch(k_to_symbol_major<__half>, grid, block, 0, st, (const __half*)src, B, n, stride_b,
                               stride_n, dst);
    case 3: return (int)launch(k_to_symbol_major<__nv_bfloat16>, grid, block, 0, st, (const __nv_bfloat16*)src, B, n,
                               stride_b, stride_n, dst);
    default: return (int)cudaErrorInvalidValue;
  }
}

int sg_from_symbol_major(const float* src, int64_t B, int64_t n, void* dst, int32_t dst_dtype, int64_t stride_b,
                         int64_t stride_n, sg_stream_t stream) {
  if (B <= 0 || n <= 0) return 0;
  dim3 block(32, 8), grid(ceil_div(B, 32), ceil_div(n, 32));
  cudaStream_t st = (cudaStream_t)stream;
  switch (dst_dtype) {
    case 0: return (int)launch(k_from_symbol_major<float>, grid, block, 0, st, src, B, n, (float*)dst, stride_b,
                               stride_n);
    case 1: return (int)launch(k_from_symbol_major<double>, grid, block, 0, st, src, B, n, (double*)dst, stride_b,
                               stride_n);
    case 2: return (int)launch(k_from_symbol_major<__half>, grid, block, 0, st, src, B, n, (__half*)dst, stride_b,
                               stride_n);
    case 3: return (int)launch(k_from_symbol_major<__nv_bfloat16>, grid, block, 0, st, src, B, n,
                               (__nv_bfloat16*)dst, stride_b, stride_n);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // extern "C"
