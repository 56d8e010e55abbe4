// DTKP-AM (top-k proofs) kernels for sm_100a.
//
// Tags are packed proof bitmasks: member u64 [rows][K][W][B], present u8 [rows][K][B].
// Ranking keys are the fp64 product of the registry probabilities of a proof's members,
// multiplied in ascending column order exactly as _dtkpcore.pyx:53-57 does, and ties are
// broken by candidate order (_dtkpcore.pyx:74-94), so retained proof sets and their row
// order are bit-identical to the CPU reference.
//
// sg_dtkp_apply fuses, per (sample, output symbol):
//   gather (provenance.py:320-326) -> conj fold with per-step normalisation
//   (provenance.py:328-341, candidate order ra*kb+rb) -> group_disj (provenance.py:352-364,
//   candidate order (ordinal-in-group, row)) into ONE streaming top-k held in registers.
// Streaming is exact: a row rejected against the running top-k can never re-enter (it has
// k distinct better rows), and a later duplicate of a retained row ranks below it.
// Long segments are cut into items whose partial top-k lists are merged by a second
// arity-1 pass of the same kernel (merging partial top-k lists is again exact).
//
// Thread mapping: lane == sample (32 samples per warp), one warp per output item; index
// records are warp-uniform, tag rows are coalesced 256-byte words per warp, the sample's
// probability column is staged in shared memory as fp64 [I][32].
#include <cstdlib>

#include "dtkp_core.cuh"

namespace sg {

static int launch_apply(const DtkpK& k, int n_blocks, cudaStream_t st) {
  switch (k.K) {
    case 1: return launch_apply_K1(k, n_blocks, st);
    case 2: return launch_apply_K2(k, n_blocks, st);
    case 3: return launch_apply_K3(k, n_blocks, st);
    case 4: return launch_apply_K4(k, n_blocks, st);
    case 5: return launch_apply_K5(k, n_blocks, st);
    case 6: return launch_apply_K6(k, n_blocks, st);
    case 7: return launch_apply_K7(k, n_blocks, st);
    case 8: return launch_apply_K8(k, n_blocks, st);
    default: return (int)cudaErrorNotSupported;
  }
}

// ------------------------------- probabilities --------------------------------------
template <int WT>
__global__ void __launch_bounds__(256) k_dtkp_probs_fwd(const uint64_t* __restrict__ member,
                                                        const uint8_t* __restrict__ present, int N, int K, int W,
                                                        const float* __restrict__ p, int I, int64_t B, int rows_per,
                                                        float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char ptile_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < B;
  const int64_t b = bval ? b0 : B - 1;
  const PCol pc = stage_pcol(ptile_raw, p, I, B, b, lane, warp, nw);
  __syncthreads();
  const int n0 = blockIdx.y * rows_per;
  const int n1 = min(N, n0 + rows_per);
  for (int n = n0 + warp; n < n1; n += nw) {
    double tot = 0.0;
    for (int q = 0; q < K; ++q) {
      if (!__ldg(present + ((size_t)n * K + q) * B + b)) continue;
      uint64_t mm[WT];
      const unsigned long long* base =
          reinterpret_cast<const unsigned long long*>(member) + ((size_t)n * K + q) * (size_t)W * B + b;
#pragma unroll
      for (int w = 0; w < WT; ++w) mm[w] = (w < W) ? __ldg(base + (size_t)w * B) : 0ull;
      tot += proof_key<WT>(mm, pc);
    }
    if (bval) out[(size_t)n * B + b] = (float)fmin(fmax(tot, 0.0), 1.0);
  }
}

// Backward of clamp(sum_r present * prod_j blended) w.r.t. p (tensor.py:302-318 rule).
// Each warp accumulates into its own fp64 [I][32] shared tile (deterministic), warps are
// summed in a fixed order and the CTA writes one partial [I][32] slab to scratch.
template <int WT>
__global__ void __launch_bounds__(128) k_dtkp_probs_bwd(const uint64_t* __restrict__ member,
                                                        const uint8_t* __restrict__ present, int N, int K, int W,
                                                        const float* __restrict__ p, int I, int64_t B, int rows_per,
                                                        const float* __restrict__ g, double* __restrict__ scratch) {
  extern __shared__ double sm[];  // ptile [I][32], then acc [nw][I][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < B;
  const int64_t b = bval ? b0 : B - 1;
  double* ptile = sm;
  double* acc = sm + (size_t)I * kWarp + (size_t)warp * I * kWarp + lane;
  for (int j = warp; j < I; j += nw) ptile[(size_t)j * kWarp + lane] = (double)__ldg(p + (size_t)j * B + b);
  for (int j = 0; j < I; ++j) acc[(size_t)j * kWarp] = 0.0;
  __syncthreads();
  const double* pl = ptile + lane;
  const int n0 = blockIdx.y * rows_per;
  const int n1 = min(N, n0 + rows_per);
  for (int n = n0 + warp; n < n1; n += nw) {
    const double gn = bval ? (double)__ldg(g + (size_t)n * B + b) : 0.0;
    for (int q = 0; q < K; ++q) {
      if (!__ldg(present + ((size_t)n * K + q) * B + b)) continue;
      uint64_t mm[WT];
      const unsigned long long* base =
          reinterpret_cast<const unsigned long long*>(member) + ((size_t)n * K + q) * (size_t)W * B + b;
#pragma unroll
      for (int w = 0; w < WT; ++w) mm[w] = (w < W) ? __ldg(base + (size_t)w * B) : 0ull;
      double prod_nz = 1.0;
      int zeros = 0;
#pragma unroll
      for (int w = 0; w < WT; ++w) {
        uint64_t x = mm[w];
        while (x) {
          const int j = __ffsll((long long)x) - 1;
          const double v = pl[(size_t)(w * 64 + j) * kWarp];
          if (v == 0.0) ++zeros; else prod_nz *= v;
          x &= x - 1;
        }
      }
      if (zeros >= 2) continue;
#pragma unroll
      for (int w = 0; w < WT; ++w) {
        uint64_t x = mm[w];
        while (x) {
          const int j = __ffsll((long long)x) - 1;
          const int col = w * 64 + j;
          const double v = pl[(size_t)col * kWarp];
          const double loo = zeros == 0 ? prod_nz / v : (v == 0.0 ? prod_nz : 0.0);
          acc[(size_t)col * kWarp] += gn * loo;
          x &= x - 1;
        }
      }
    }
  }
  __syncthreads();
  // fixed-order reduction over warps, one [I][32] slab per CTA
  double* slab = scratch + (size_t)blockIdx.y * I * B;
  for (int j = warp; j < I; j += nw) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += sm[(size_t)I * kWarp + ((size_t)w * I + j) * kWarp + lane];
    if (bval) slab[(size_t)j * B + b0] = s;
  }
}

__global__ void k_reduce_slabs(const double* __restrict__ scratch, int n_slabs, int64_t n_elem,
                               float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_elem; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < n_slabs; ++c) s += scratch[(size_t)c * n_elem + i];
    out[i] = (float)s;
  }
}

// Rows per CTA so that a probs launch is ~4 waves of 148 SMs.
static int probs_rows_per(int N, int64_t B, int nw) {
  const int tiles_b = ceil_div(B, kWarp);
  int chunks = ceil_div(148 * 4, tiles_b);
  if (chunks < 1) chunks = 1;
  int rows = ceil_div(N, chunks);
  if (rows < nw) rows = nw;
  return rows;
}

static int bwd_warps(int I) {
  // shared: ptile I*32*8 + nw * I*32*8 <= 200 KB
  const size_t per = (size_t)I * kWarp * sizeof(double);
  int nw = 4;
  while (nw > 1 && per * (nw + 1) > 200 * 1024) --nw;
  return nw;
}

// ------------------------------- dedup_topk (drop-in) -------------------------------
template <int K, int WT>
__global__ void __launch_bounds__(128) k_dedup_topk(const uint8_t* __restrict__ member,
                                                    const uint8_t* __restrict__ present, const double* __restrict__ p,
                                                    int64_t M, int R, int I, int k, uint8_t* __restrict__ out_member,
                                                    uint8_t* __restrict__ out_present) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (int64_t)gridDim.x * blockDim.x) {
    TopK<K, WT> S;
    S.clear();
    const double* pm = p + (size_t)m * I;
    for (int r = 0; r < R; ++r) {
      if (!present[(size_t)m * R + r]) continue;
      const uint8_t* row = member + ((size_t)m * R + r) * I;
      uint64_t mm[WT];
#pragma unroll
      for (int w = 0; w < WT; ++w) mm[w] = 0ull;
      double prob = 1.0;
      for (int j = 0; j < I; ++j) {
        if (row[j]) {
#pragma unroll
          for (int w = 0; w < WT; ++w)
            if (w == (j >> 6)) mm[w] |= 1ull << (j & 63);
          prob *= pm[j];
        }
      }
      S.insert(mm, prob, r);
    }
    for (int a2 = 0; a2 < k; ++a2) {
      uint8_t* dst = out_member + ((size_t)m * k + a2) * I;
      if (a2 < S.n) {
        int src = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
          if (i == a2) src = S.idx[i];
        const uint8_t* row = member + ((size_t)m * R + src) * I;
        for (int j = 0; j < I; ++j) dst[j] = row[j];
        out_present[(size_t)m * k + a2] = 1;
      } else {
        for (int j = 0; j < I; ++j) dst[j] = 0;
        out_present[(size_t)m * k + a2] = 0;
      }
    }
  }
}

template <int K>
static int dedup_k(const uint8_t* member, const uint8_t* present, const double* p, int64_t M, int R, int I, int k,
                   uint8_t* om, uint8_t* op, cudaStream_t st) {
  const int W = (I + 63) / 64;
  int grid = ceil_div(M, 128);
  if (grid > 4096) grid = 4096;
  if (W > 8) return (int)cudaErrorNotSupported;
  count_launch();
  if (W <= 1)
    k_dedup_topk<K, 1><<<grid, 128, 0, st>>>(member, present, p, M, R, I, k, om, op);
  else if (W <= 2)
    k_dedup_topk<K, 2><<<grid, 128, 0, st>>>(member, present, p, M, R, I, k, om, op);
  else if (W <= 4)
    k_dedup_topk<K, 4><<<grid, 128, 0, st>>>(member, present, p, M, R, I, k, om, op);
  else
    k_dedup_topk<K, 8><<<grid, 128, 0, st>>>(member, present, p, M, R, I, k, om, op);
  SG_LAUNCH_CHECK();
  return 0;
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_dtkp_apply(const sg_dtkp_apply_desc* d, sg_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  SG_RETURN_IF(d->arity < 1 || d->arity > SG_MAX_ARITY, cudaErrorInvalidValue);
  SG_RETURN_IF(d->K < 1 || d->K > 8 || d->W > 8, cudaErrorNotSupported);
  if (d->B <= 0 || d->seg.n_seg <= 0) return 0;
  DtkpK k{};
  for (int i = 0; i < d->arity; ++i) k.ops[i] = d->ops[i];
  k.tail = d->op_tail;
  k.arity = d->arity;
  k.K = d->K;
  k.W = d->W;
  k.I = d->I;
  k.B = d->B;
  k.p = d->p;
  k.recs = d->seg.recs;
  k.rec_words = d->seg.rec_words;
  k.items = d->seg.items;
  k.blk = d->seg.blk;
  k.out_m = d->out_member;
  k.out_p = d->out_present;
  k.scr_m = d->scratch_member;
  k.scr_p = d->scratch_present;
  k.sched = d->sched;
  k.n_items = d->seg.n_items;
  k.fused = 0;
  k.packed = d->seg_packed;
  k.ranked = d->rows_ranked;
  if (d->inner_arity != 0) {
    // fused conj -> group_disj: only an arity-1 apply over a binary conj
    SG_RETURN_IF(d->arity != 1 || d->inner_arity != 2 || d->seg.rec_words < 2, cudaErrorInvalidValue);
    k.inner[0] = d->inner_ops[0];
    k.inner[1] = d->inner_ops[1];
    k.fused = 1;
  }
  if (d->seg.n_items > 0) {
    int rc = launch_apply(k, d->seg.n_blocks, st);
    if (rc) return rc;
  }
  if (d->seg.n_split > 0) {
    DtkpK m = k;
    m.arity = 1;
    m.fused = 0;  // merges read the materialised partial lists
    m.packed = 0;
    m.ranked = 1;  // partial lists are written in rank order
    m.ops[0].member = d->scratch_member;
    m.ops[0].present = d->scratch_present;
    m.ops[0].rows = d->seg.n_partial;
    m.ops[0].W = d->W;
    m.tail = m.ops[0];
    m.recs = d->merge.recs;
    m.rec_words = d->merge.rec_words;
    m.items = d->merge.items;
    m.blk = d->merge.blk;
    m.n_items = d->merge.n_items;
    const bool two = d->merge.n_split > 0;
    SG_RETURN_IF(two && (d->scratch2_member == nullptr || d->scratch2_present == nullptr), cudaErrorInvalidValue);
    m.scr_m = two ? d->scratch2_member : nullptr;
    m.scr_p = two ? d->scratch2_present : nullptr;
    int rc = launch_apply(m, d->merge.n_blocks, st);
    if (rc) return rc;
    if (two) {  // second level: the split merge segments' partial lists -> the output rows
      DtkpK m2 = m;
      m2.ops[0].member = d->scratch2_member;
      m2.ops[0].present = d->scratch2_present;
      m2.ops[0].rows = d->merge.n_partial;
      m2.tail = m2.ops[0];
      m2.recs = d->merge2.recs;
      m2.rec_words = d->merge2.rec_words;
      m2.items = d->merge2.items;
      m2.blk = d->merge2.blk;
      m2.n_items = d->merge2.n_items;
      m2.scr_m = nullptr;
      m2.scr_p = nullptr;
      rc = launch_apply(m2, d->merge2.n_blocks, st);
      if (rc) return rc;
    }
  }
  return 0;
}

int sg_dtkp_probs_fwd(const uint64_t* member, const uint8_t* present, int32_t N, int32_t K, int32_t W, const float* p,
                      int32_t I, int64_t B, float* out, sg_stream_t stream) {
  if (N <= 0 || B <= 0) return 0;
  SG_RETURN_IF(W > 8, cudaErrorNotSupported);
  cudaStream_t st = (cudaStream_t)stream;
  const int nw = 8;
  const int rows_per = probs_rows_per(N, B, nw);
  dim3 grid(ceil_div(B, kWarp), ceil_div(N, rows_per));
  const int mode = ptile_mode(I);
  SG_RETURN_IF(mode == 0, cudaErrorNotSupported);
  const size_t smem = ptile_bytes(I);
#define SG_PF(WT)                                                                                        \
  do {                                                                                                   \
    ensure_smem((const void*)k_dtkp_probs_fwd<WT>, smem);                                                \
    count_launch();                                                                                      \
    k_dtkp_probs_fwd<WT><<<grid, nw * 32, smem, st>>>(member, present, N, K, W, p, I, B, rows_per, out);  \
  } while (0)
  if (W <= 1) SG_PF(1);
  else if (W <= 2) SG_PF(2);
  else if (W <= 4) SG_PF(4);
  else SG_PF(8);
#undef SG_PF
  SG_LAUNCH_CHECK();
  return 0;
}

int64_t sg_dtkp_probs_bwd_scratch(int32_t N, int32_t I, int64_t B) {
  if (N <= 0 || B <= 0 || I <= 0) return 0;
  const int nw = bwd_warps(I);
  const int rows_per = probs_rows_per(N, B, nw);
  const int chunks = ceil_div(N, rows_per);
  return (int64_t)chunks * I * B * (int64_t)sizeof(double);
}

int sg_dtkp_probs_bwd(const uint64_t* member, const uint8_t* present, int32_t N, int32_t K, int32_t W, const float* p,
                      int32_t I, int64_t B, const float* grad_out, float* grad_p, void* scratch, sg_stream_t stream) {
  if (B <= 0 || I <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (N <= 0) {
    cudaError_t e = cudaMemsetAsync(grad_p, 0, (size_t)I * B * sizeof(float), st);
    return (int)e;
  }
  SG_RETURN_IF(W > 8, cudaErrorNotSupported);
  const int nw = bwd_warps(I);
  const size_t smem = (size_t)I * kWarp * sizeof(double) * (nw + 1);
  SG_RETURN_IF(smem > 227 * 1024, cudaErrorNotSupported);
  const int rows_per = probs_rows_per(N, B, nw);
  const int chunks = ceil_div(N, rows_per);
  dim3 grid(ceil_div(B, kWarp), chunks);
  double* scr = (double*)scratch;
#define SG_PB(WT)                                                                                                  \
  do {                                                                                                             \
    ensure_smem((const void*)k_dtkp_probs_bwd<WT>, smem);                                                          \
    count_launch();                                                                                      \
    k_dtkp_probs_bwd<WT><<<grid, nw * 32, smem, st>>>(member, present, N, K, W, p, I, B, rows_per, grad_out, scr); \
  } while (0)
  if (W <= 1) SG_PB(1);
  else if (W <= 2) SG_PB(2);
  else if (W <= 4) SG_PB(4);
  else SG_PB(8);
#undef SG_PB
  SG_LAUNCH_CHECK();
  const int64_t n_elem = (int64_t)I * B;
  int g2 = ceil_div(n_elem, 256);
  if (g2 > 148 * 8) g2 = 148 * 8;
  count_launch();
  k_reduce_slabs<<<g2, 256, 0, st>>>(scr, chunks, n_elem, grad_p);
  SG_LAUNCH_CHECK();
  return 0;
}

int sg_dedup_topk(const uint8_t* member, const uint8_t* present, const double* p, int64_t M, int32_t R, int32_t I,
                  int32_t k, uint8_t* out_member, uint8_t* out_present, sg_stream_t stream) {
  if (M <= 0 || k <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (R <= 0) {
    cudaError_t e = cudaMemsetAsync(out_member, 0, (size_t)M * k * (I > 0 ? I : 0), st);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaMemsetAsync(out_present, 0, (size_t)M * k, st);
  }
  SG_RETURN_IF(I > 512, cudaErrorNotSupported);
  switch (k) {
    case 1: return dedup_k<1>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 2: return dedup_k<2>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 3: return dedup_k<3>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 4: return dedup_k<4>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 5: return dedup_k<5>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 6: return dedup_k<6>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 7: return dedup_k<7>(member, present, p, M, R, I, k, out_member, out_present, st);
    case 8: return dedup_k<8>(member, present, p, M, R, I, k, out_member, out_present, st);
    default: return (int)cudaErrorNotSupported;
  }
}

}  // extern "C"
