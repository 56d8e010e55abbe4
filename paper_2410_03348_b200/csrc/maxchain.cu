// Fused max-product Toeplitz chains (the north star's max/DAMP variant) for sm_100a.
//
// A left fold of max-product applies v_i = clamp01(max-prod(v_{i-1}, S_i)), where every
// step is apply(f, res, d_i) with T[s][j] = s + j and the long operand first (every
// sum_n fold step, programs.py:42-49, under DampMax), runs as ONE forward and ONE
// backward launch instead of m generic sg_maxprod launches each way.  Per step the
// arithmetic is exactly sg_maxprod_fwd/bwd's (maxprod.cu): the records of output o are
// (s, o - s) in enumeration order (s ascending), value = max of the fp32 products with the
// FIRST maximal record kept (tensor.py:319-325), clamp01 after; the backward sends g[o] to
// that record only, and every gradient row is the fmaf sum of its contributions in record
// order (input row s: o ascending; filter row j: s ascending) — bit-identical to the
// per-apply kernels.
//
// Mapping.  Lane = sample: a sample's whole chain lives in its own shared-memory column,
// so no two lanes ever touch the same word and the kernels need no barrier at all.  The
// forward updates the state in place (outputs descending, four at a time from one
// 13-row window), streams the clamped intermediate states to HBM row-major over the batch
// and the argmax tap j* (one byte per step, output, sample) packed four outputs to a
// 32-bit word in a warp-blocked layout ([warp][word][32 lanes]: one coalesced 128-byte
// access per four outputs of the warp).  The
// backward walks the steps down, loads v_{i-1} into its column, and scatters each
// output's upstream gradient to its argmax record: G_{i-1}[s*] += g[o] * S[j*] (shared
// column) and dS[j*] += g[o] * v_{i-1}[s*] (registers, select-updated), o ascending.
#include "common.cuh"

namespace sg {

constexpr int kMcMaxSteps = 32;

__device__ __forceinline__ void mc_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct MCRows {
  const float* p;
  int64_t sr, sb;
  __device__ __forceinline__ float ld(int64_t r, int64_t b) const { return __ldg(p + r * sr + b * sb); }
};

struct MaxChainArgs {
  MCRows base;
  MCRows filt[kMcMaxSteps];
  float* dfilt_p[kMcMaxSteps];
  int64_t dfilt_sr[kMcMaxSteps], dfilt_sb[kMcMaxSteps];
  int n[kMcMaxSteps + 1];
  int state_off[kMcMaxSteps + 1];  // row offset of v_i (i = 1..m-1) in `states`
  int arg_off[kMcMaxSteps + 1];    // word offset of step i's packed argmax (4 outputs per word)
  int arg_words;                   // packed argmax words per warp
  int m, n_max;
  int64_t B;
  float* states;         // [state rows][B]
  uint32_t* argmax;      // [warp][arg_words][32]: byte k of word w = j* of output 4w + k of the step
  float* out;            // [n_m][B]
  double* rowsum;        // optional [B]
  const float* g_out;    // [n_m][B]
  float* dbase_p;
  int64_t dbase_sr, dbase_sb;
};

template <int KF>
__device__ __forceinline__ void maxrec(float& best, int& arg, float v, int j, bool valid) {
  // records arrive s ascending (j descending): the first valid one seeds, later ones replace
  // only when strictly greater — the first maximal record wins (maxprod.cu)
  if (valid && (arg < 0 || v > best)) {
    best = v;
    arg = j;
  }
}

// Forward.  P lanes share one sample (SPW = 32 / P samples per warp): the state of sample
// c ping-pongs between two shared columns (stride SPW floats, KF-1 zero rows in front), and
// the lanes of a sample take the step's output groups of four round-robin, so a step's
// dependent compare/select chains are split P ways (the kernel is bound by them: one warp
// per scheduler at P = 1); one __syncwarp per step.  Each output is computed exactly as
// before (same records, same order, same first-maximal rule), so P does not change a bit.
template <int KF, int P>
__global__ void __launch_bounds__(32) k_maxchain_fwd(const MaxChainArgs a) {
  extern __shared__ float mcs[];
  constexpr int SPW = 32 / P;
  constexpr int PAD = KF - 1;
  const int lane = threadIdx.x;
  const int c = lane % SPW, h = lane / SPW;
  const int64_t b0 = (int64_t)blockIdx.x * SPW + c;
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  const int rows = PAD + a.n_max;
  float* const VA = mcs + c;  // buffer 0 of sample c: row r at VA[r * SPW]; buffer 1 after it
  float* const VB = VA + (size_t)rows * SPW;
  mc_pdl_wait();
  for (int r = h; r < PAD; r += P) {
    VA[r * SPW] = 0.f;
    VB[r * SPW] = 0.f;
  }
  for (int r = h; r < a.n[0]; r += P) VA[(PAD + r) * SPW] = a.base.ld(r, b);
  float fn[KF];  // the next step's filter, loaded one step ahead
#pragma unroll
  for (int j = 0; j < KF; ++j) fn[j] = a.filt[0].ld(j, b);
  // argmax bytes: [32-sample block][word][32 lanes], byte (o & 3) of word o >> 2
  uint8_t* const am = reinterpret_cast<uint8_t*>(a.argmax + (size_t)(b0 >> 5) * a.arg_words * 32 + (b0 & 31));
  __syncwarp();
  for (int i = 1; i <= a.m; ++i) {
    float f[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) f[j] = fn[j];
    if (i < a.m) {
#pragma unroll
      for (int j = 0; j < KF; ++j) fn[j] = a.filt[i].ld(j, b);
    }
    const int nin = a.n[i - 1], nout = a.n[i];
    const bool last = i == a.m;
    const float* Vin = (i & 1) ? VA : VB;
    float* Vout = (i & 1) ? VB : VA;
    float* gst = last ? a.out : a.states + (size_t)a.state_off[i] * a.B;
    uint8_t* gam = am + (size_t)a.arg_off[i] * 128;
    // output groups o0 - 3 .. o0 (o0 = nout - 1 - 4 gi), one window of KF + 3 rows each
    for (int o0 = nout - 1 - 4 * h; o0 >= 0; o0 -= 4 * P) {
      float w[KF + 3];
#pragma unroll
      for (int u = 0; u < KF + 3; ++u) {
        const int s = o0 - 3 - PAD + u;  // s >= -PAD - 3; rows < -PAD read as 0 (masked below)
        w[u] = s >= -PAD ? Vin[(PAD + s) * SPW] : 0.f;
      }
      float best[4];
      int arg[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        best[q] = 0.f;
        arg[q] = -1;
      }
#pragma unroll
      for (int j = KF - 1; j >= 0; --j) {  // s = o - j ascending
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int o = o0 - q;
          const int s = o - j;
          maxrec<KF>(best[q], arg[q], w[3 - q + PAD - j] * f[j], j, o >= 0 && s >= 0 && s < nin);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int o = o0 - q;
        if (o < 0) break;
        const float v = clamp01(best[q]);  // every output of a Toeplitz step has a record
        Vout[(PAD + o) * SPW] = v;
        if (bval) {
          gst[(size_t)o * a.B + b0] = v;
          gam[(size_t)(o >> 2) * 128 + (o & 3) * 1] = (uint8_t)arg[q];
        }
      }
    }
    __syncwarp();
  }
  if (a.rowsum != nullptr && bval && h == 0) {
    // outputs descending, as the one-lane-per-sample forward summed them
    const float* Vl = (a.m & 1) ? VB : VA;
    double rs = 0.0;
    for (int o = a.n[a.m] - 1; o >= 0; --o) rs += (double)Vl[(PAD + o) * SPW];
    a.rowsum[b0] = rs;
  }
}

__device__ __forceinline__ void mc_cp4(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void mc_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void mc_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Backward.  Columns: G (the upstream gradient, updated IN PLACE into the next one) and
// V[2] (v_{i-1} of the current step and, arriving through cp.async while this step runs,
// v_{i-2} of the next).  In place: output o is read at iteration o and its slot restarts
// as the accumulator of input row o (every contribution to input row s comes from an
// output o >= s, o ascending), so the new gradient never overwrites an unread one.
template <int KF>
__global__ void __launch_bounds__(32) k_maxchain_bwd(const MaxChainArgs a) {
  extern __shared__ float mcs[];
  const int lane = threadIdx.x;
  const int64_t b0 = (int64_t)blockIdx.x * 32 + lane;
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  float* G = mcs + lane;
  float* const V0 = G + (size_t)a.n_max * 32;  // buffer t at V0 + t * col
  const size_t col = (size_t)a.n_max * 32;
  // v_{i-1} rows -> column Vd (i >= 1): the stored state, or the base operand for i = 1
  auto stage_prev = [&](float* Vd, int i) {
    const int nin = a.n[i - 1];
    if (i > 1) {
      const float* st = a.states + (size_t)a.state_off[i - 1] * a.B + b;
      for (int s = 0; s < nin; ++s) mc_cp4(Vd + s * 32, st + (size_t)s * a.B);
    } else {
      for (int s = 0; s < nin; ++s) mc_cp4(Vd + s * 32, a.base.p + s * a.base.sr + b * a.base.sb);
    }
  };
  mc_pdl_wait();
  for (int o = 0; o < a.n[a.m]; ++o) mc_cp4(G + o * 32, a.g_out + (size_t)o * a.B + b);
  stage_prev(V0, a.m);
  mc_commit();
  float fn[KF];  // the next (lower) step's filter, loaded one step ahead
#pragma unroll
  for (int j = 0; j < KF; ++j) fn[j] = a.filt[a.m - 1].ld(j, b);
  // packed argmax taps, 32 outputs (8 words) per batch, loaded one batch ahead (across
  // step boundaries too)
  constexpr int kBatch = 32;
  auto load_words = [&](uint32_t (&jw)[kBatch / 4], int i, int o0) {
    const uint32_t* am = a.argmax + ((size_t)blockIdx.x * a.arg_words + a.arg_off[i]) * 32 + lane;
#pragma unroll
    for (int q = 0; q < kBatch / 4; ++q)  // lanes past B read tap 0 (their bytes are never written)
      jw[q] = bval && o0 + 4 * q < a.n[i] ? __ldg(am + (size_t)((o0 >> 2) + q) * 32) : 0u;
  };
  uint32_t jn[kBatch / 4];
  load_words(jn, a.m, 0);
  for (int i = a.m; i >= 1; --i) {
    const int nout = a.n[i];
    float* Vp = V0 + ((a.m - i) & 1) * col;
    float f[KF], dS[KF];
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      f[j] = fn[j];
      dS[j] = 0.f;
    }
    if (i > 1) {
#pragma unroll
      for (int j = 0; j < KF; ++j) fn[j] = a.filt[i - 2].ld(j, b);
      stage_prev(V0 + ((a.m - i + 1) & 1) * col, i - 1);  // the next step's v_{i-2}, in flight during this step
    }
    mc_commit();
    mc_wait<1>();  // this step's rows (and, at the top, G) have landed; the newest group may fly
    for (int o0 = 0; o0 < nout; o0 += kBatch) {
      uint32_t jw[kBatch / 4];
#pragma unroll
      for (int q = 0; q < kBatch / 4; ++q) jw[q] = jn[q];
      if (o0 + kBatch < nout)
        load_words(jn, i, o0 + kBatch);
      else if (i > 1)
        load_words(jn, i - 1, 0);
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        const int o = o0 + q;
        if (o >= nout) break;
        const int j = (int)((jw[q >> 2] >> (8 * (q & 3))) & 0xffu);  // byte (o & 3) of word o >> 2
        const int s = o - j;
        const float g = G[o * 32];
        G[o * 32] = 0.f;  // slot o now accumulates input row o
        float fj = f[0];
#pragma unroll
        for (int jj = 1; jj < KF; ++jj) fj = jj == j ? f[jj] : fj;
        G[s * 32] = fmaf(g, fj, G[s * 32]);
        const float vs = Vp[s * 32];
#pragma unroll
        for (int jj = 0; jj < KF; ++jj) dS[jj] = jj == j ? fmaf(g, vs, dS[jj]) : dS[jj];
      }
    }
    if (bval) {
#pragma unroll
      for (int j = 0; j < KF; ++j) a.dfilt_p[i - 1][j * a.dfilt_sr[i - 1] + b0 * a.dfilt_sb[i - 1]] = dS[j];
    }
  }
  if (bval)
    for (int s = 0; s < a.n[0]; ++s) a.dbase_p[s * a.dbase_sr + b0 * a.dbase_sb] = G[s * 32];
}

static int mc_fill(MaxChainArgs& a, const sg_chain* c) {
  if (c->m < 1 || c->m > kMcMaxSteps || c->kf < 1 || c->kf > 16 || c->n0 < 1) return (int)cudaErrorInvalidValue;
  a.base = MCRows{c->base.ptr, c->base.stride_row, c->base.stride_b};
  a.m = c->m;
  a.B = c->B;
  a.n[0] = c->n0;
  int soff = 0, aoff = 0, nmax = c->n0;
  for (int i = 1; i <= c->m; ++i) {
    a.n[i] = a.n[i - 1] + c->kf - 1;
    a.filt[i - 1] = MCRows{c->filters[i - 1].ptr, c->filters[i - 1].stride_row, c->filters[i - 1].stride_b};
    a.state_off[i] = soff;
    if (i < c->m) soff += a.n[i];
    a.arg_off[i] = aoff;
    aoff += (a.n[i] + 3) / 4;
    if (a.n[i] > nmax) nmax = a.n[i];
  }
  a.state_off[0] = a.arg_off[0] = 0;
  a.arg_words = aoff;
  a.n_max = nmax;
  a.states = c->states;
  return 0;
}

template <typename... KArgs>
static cudaError_t mc_launch(void (*kernel)(KArgs...), const MaxChainArgs& a, size_t smem, cudaStream_t st,
                             int spw = 32) {
  cudaError_t e = ensure_smem((const void*)kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ceil_div(a.B, spw));
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

#define SG_MC_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

}  // namespace sg

using namespace sg;

extern "C" {

int64_t sg_maxchain_states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B) {
  int64_t rows = 0, n = n0;
  for (int i = 1; i < m; ++i) {
    n += kf - 1;
    rows += n;
  }
  return rows * B;
}

int64_t sg_maxchain_argmax_bytes(int32_t n0, int32_t kf, int32_t m, int64_t B) {
  int64_t words = 0, n = n0;
  for (int i = 1; i <= m; ++i) {
    n += kf - 1;
    words += (n + 3) / 4;
  }
  return words * 4 * 32 * ((B + 31) / 32);  // [warp][words][32 lanes] u32
}

int32_t sg_maxchain_max_rows(int32_t kf) {
  if (kf < 1 || kf > 16) return 0;
  // backward: three columns (G, two v_{i-1} buffers) of n_max rows x 32 lanes x 4 B
  return (int32_t)(227 * 1024 / (3 * 32 * 4));
}

int sg_maxchain_fwd(const sg_chain* c, float* out, double* rowsum, uint8_t* argmax, sg_stream_t stream) {
  MaxChainArgs a{};
  int rc = mc_fill(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  SG_RETURN_IF(a.n_max > sg_maxchain_max_rows(c->kf), cudaErrorNotSupported);
  a.out = out;
  a.rowsum = rowsum;
  a.argmax = reinterpret_cast<uint32_t*>(argmax);
  SG_RETURN_IF(((uintptr_t)argmax & 3) != 0, cudaErrorInvalidValue);
  // lanes per sample: enough warps to give every scheduler ~4 of them (the forward is
  // bound by its per-lane compare/select chains), P = 4 up to B ~ 19k
  int P = 4;
  if (const char* e = getenv("SG_MC_LANES")) P = atoi(e);
  else if (c->B > 37888) P = 1;
  else if (c->B > 18944) P = 2;
  SG_RETURN_IF(P != 1 && P != 2 && P != 4, cudaErrorInvalidValue);
  // two state columns per sample, 32 columns-per-buffer-pair per warp whatever P is
  const size_t smem = (size_t)2 * (c->kf - 1 + a.n_max) * 32 * sizeof(float);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K)                                                                               \
  case K:                                                                                  \
    return (int)(P == 4   ? mc_launch(k_maxchain_fwd<K, 4>, a, smem / 4, st, 8)            \
                 : P == 2 ? mc_launch(k_maxchain_fwd<K, 2>, a, smem / 2, st, 16)           \
                          : mc_launch(k_maxchain_fwd<K, 1>, a, smem, st, 32));
    SG_MC_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

int sg_maxchain_bwd(const sg_chain* c, const uint8_t* argmax, const float* grad_out, sg_rows grad_base,
                    const sg_rows* grad_filters, sg_stream_t stream) {
  MaxChainArgs a{};
  int rc = mc_fill(a, c);
  if (rc) return rc;
  if (c->B <= 0) return 0;
  SG_RETURN_IF(a.n_max > sg_maxchain_max_rows(c->kf), cudaErrorNotSupported);
  a.argmax = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(argmax));
  SG_RETURN_IF(((uintptr_t)argmax & 3) != 0, cudaErrorInvalidValue);
  a.g_out = grad_out;
  a.dbase_p = grad_base.ptr;
  a.dbase_sr = grad_base.stride_row;
  a.dbase_sb = grad_base.stride_b;
  for (int i = 0; i < c->m; ++i) {
    a.dfilt_p[i] = grad_filters[i].ptr;
    a.dfilt_sr[i] = grad_filters[i].stride_row;
    a.dfilt_sb[i] = grad_filters[i].stride_b;
  }
  const size_t smem = (size_t)3 * a.n_max * 32 * sizeof(float);
  cudaStream_t st = (cudaStream_t)stream;
  switch (c->kf) {
#define X(K) \
  case K: return (int)mc_launch(k_maxchain_bwd<K>, a, smem, st);
    SG_MC_CASES(X)
#undef X
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // extern "C"
