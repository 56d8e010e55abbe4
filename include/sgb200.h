/*
 * sgb200.h — C ABI of the B200-native Dolphin probabilistic hot path.
 *
 * Every entry point:
 *   - returns 0 on success or a cudaError_t value (never throws across the ABI);
 *   - takes CALLER-ALLOCATED DEVICE buffers (the PyTorch caching allocator owns them);
 *   - enqueues work on the given cudaStream_t and never synchronises the host;
 *   - has no global mutable state (re-entrant; use distinct streams per thread);
 *   - has no CPU fallback: if the device code is missing the call fails.
 *
 * Tag layouts in HBM (symbol-major, batch innermost, so lane == sample is coalesced):
 *   DAMP tags      float    [rows][B]
 *   DTKP members   uint64   [rows][K][W][B]   bit j of word w = input column 64*w + j
 *   DTKP present   uint8    [rows][K][B]
 *   registry probs float    [I][B]
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/symgrad/):
 *   sg_damp_apply_fwd   provenance.py:233 gather + :236 conj fold + :242-253 group_disj
 *                       (distribution.py:262-270 tag work of apply_if)
 *   sg_damp_apply_bwd   tensor.py:287 clamp bw, :415 affine bw, :240 mul bw, :386-391 select_rows bw
 *   sg_segsum_run       provenance.py:242-253 Damp.group_disj (and select_rows bw scatter-add)
 *   sg_damp_rows_add    provenance.py:239-240 Damp.disj; distribution.py:279-297 union
 *   sg_chain_fwd/bwd    a left fold of Toeplitz applies (programs.py:42-49 sum_n) as one
 *                       launch each way; per step the same as sg_damp_apply_fwd/bwd
 *   sg_maxchain_fwd/bwd the same fold under the max/DAMP variant (per step sg_maxprod_*)
 *   sg_nll_fwd/bwd      learn.py:92-119 loss_nll (the caller right after get_probs)
 *   sg_rows_gather      provenance.py:233-234 / :320-326 gather (filter, distribution.py:158-169)
 *   sg_to_symbol_major  provenance.py:223-225 Damp.input_tags (layout + fp32 cast of the block)
 *   sg_dtkp_apply       provenance.py:328-341 conj, :343-350 disj, :352-364 group_disj,
 *                       :366-379 _normalize (fused streaming top-k, bit-exact ranking)
 *   sg_dtkp_probs_fwd   provenance.py:398-413 DtkpAm.probs / :415-423 forward_probs
 *   sg_dtkp_probs_bwd   tensor.py:302-318 reduce_prod leave-one-out bw (+ clamp/sum/mul bw)
 *   sg_dedup_topk       _dtkpcore.pyx:17-96 dedup_topk (kernels.py:29-42 dispatch) — same
 *                       argument meaning, byte layout and ordering semantics
 */
#ifndef SGB200_H
#define SGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sg_stream_t; /* == cudaStream_t */

#define SG_MAX_ARITY 8

/* One segmented sum-of-products problem:
 *   out[seg][b] = (clamp?)  sum_{rec in seg}  prod_{i < n_ops}  op_i[ recs[rec][i] ][b]
 * Segments are cut into items of bounded length; a segment cut into several items
 * writes partial rows into `scratch` and is finished by a deterministic fix-up pass. */
typedef struct sg_segsum {
  int32_t n_seg;      /* output rows                                            */
  int32_t rec_words;  /* int32 words per record: 1, 2, 4 or 8 (>= n_ops)         */
  int32_t n_items;    /* work items                                             */
  int32_t n_blocks;   /* CTA chunks along grid.y                                */
  int32_t n_split;    /* segments spread over more than one item                */
  int32_t n_partial;  /* partial rows needed in scratch ([n_partial][B] floats)  */
  int32_t staged;     /* 1: stage operand tiles in shared memory                */
  int32_t n_recs;     /* records (rows of recs)                                 */
  const int32_t* recs;  /* [n_recs][rec_words]                                  */
  const int32_t* items; /* [n_items][4] = seg, rec_begin, rec_end, dest (-1 = direct) */
  const int32_t* blk;   /* [n_blocks + 1] item range of each CTA chunk            */
  const int32_t* split; /* [n_split][3] = seg, partial_begin, partial_end          */
} sg_segsum;

/* A memoised apply plan (host-built from the black-box symbol function). */
typedef struct sg_damp_plan {
  int32_t arity;
  int32_t n_out;
  int32_t sizes[SG_MAX_ARITY];
  int32_t conv;        /* Toeplitz tables (f = sum of the input positions, no drops):
                        * 1: arity 2, one side <= 16 symbols (register-filter kernels);
                        * 2: arity 2, both sides long (direct per-sample convolution);
                        * 3: arity 3, run as (in0 (*) in1) (*) in2 — needs scratch of
                        *    (sizes[0] + sizes[1] - 1) x B floats forward, twice that backward;
                        * 0: anything else (segmented sum-of-products plans below)       */
  int32_t conv_short;  /* conv == 1: which input (0/1) is the short "filter" side        */
  sg_segsum fwd;              /* segments = output symbols, records = input positions   */
  sg_segsum bwd[SG_MAX_ARITY];/* segments = positions of input k, records = (T[c], s_j!=k) */
} sg_damp_plan;

int sg_version(void);
/* Kernels this library has enqueued so far (all entry points; graph capture counts once). */
int64_t sg_launch_count(void);
int sg_device_sm_count(int device);

/* ---- layout: user (B, n) block  <->  symbol-major [n][B] fp32 ----------------------
 * dtype codes: 0 = float32, 1 = float64, 2 = float16, 3 = bfloat16 (strides in elements) */
int sg_to_symbol_major(const void* src, int32_t src_dtype, int64_t B, int64_t n,
                       int64_t stride_b, int64_t stride_n, float* dst, sg_stream_t stream);
int sg_from_symbol_major(const float* src, int64_t B, int64_t n, void* dst, int32_t dst_dtype,
                         int64_t stride_b, int64_t stride_n, sg_stream_t stream);

/* A strided fp32 [rows][B] operand: element (r, b) lives at ptr[r * stride_row + b * stride_b].
 * Symbol-major tags have (B, 1); a user (B, n) row-major block is read in place with (1, n);
 * stride_b == 0 broadcasts a batch-1 operand (forward only). */
typedef struct sg_rows {
  float* ptr;
  int64_t stride_row;
  int64_t stride_b;
} sg_rows;

/* ---- DAMP (add-mult) --------------------------------------------------------------- */
int sg_segsum_run(const sg_segsum* prob, const sg_rows* ops, const int32_t* op_rows,
                  int32_t n_ops, int64_t B, int32_t clamp01, sg_rows out, float* scratch,
                  sg_stream_t stream);
/* out: contiguous [n_out][B]; scratch: [fwd.n_partial][B] floats (may be NULL if 0). */
int sg_damp_apply_fwd(const sg_damp_plan* plan, const sg_rows* inputs, int64_t B,
                      float* out, float* scratch, sg_stream_t stream);
/* grad_out: [n_out][B] rows with any strides (the short-filter Toeplitz path, conv == 1,
 * needs stride_b == 1 and stride_row == B); grad_in[k].ptr == NULL skips input k (conv == 1
 * needs both); scratch: [max_k bwd[k].n_partial][B] floats. */
int sg_damp_apply_bwd(const sg_damp_plan* plan, const sg_rows* inputs,
                      sg_rows grad_out, int64_t B, const sg_rows* grad_in,
                      float* scratch, sg_stream_t stream);
/* out[r][b] = clamp01(A[ia[r]][b] + Bm[ib[r]][b]) into contiguous [n_rows][B];
 * index -1 contributes 0. */
int sg_damp_rows_add(const sg_rows A, const int32_t* ia, const sg_rows Bm, const int32_t* ib,
                     int64_t n_rows, int64_t B, int32_t clamp01, float* out, sg_stream_t stream);

/* ---- max-product apply (the north star's "max/DAMP variant") ----------------------
 * conj = product (left to right), disj = max over the output's records with the gradient
 * to the FIRST maximal record (tensor.py:319-325 reduce "max"); empty output = 0;
 * optional clamp01 after the max (gradient passes through).  Records of output s are
 * recs[seg_off[s] .. seg_off[s+1]) in first-derivation order; rec_out[c] is the output
 * of record c; in_off[k] / in_recs[k] list, per row of input k, the records that use it
 * (ascending).  The backward writes (overwrites) grad_in[k] for every non-NULL entry. */
typedef struct sg_maxprod_plan {
  int32_t arity;
  int32_t n_out;
  int32_t n_recs;
  int32_t sizes[SG_MAX_ARITY];
  const int32_t* seg_off;                /* [n_out + 1]        */
  const int32_t* recs;                   /* [n_recs][arity]    */
  const int32_t* rec_out;                /* [n_recs]           */
  const int32_t* in_off[SG_MAX_ARITY];   /* [sizes[k] + 1]     */
  const int32_t* in_recs[SG_MAX_ARITY];  /* [n_recs]           */
} sg_maxprod_plan;

/* out, argmax: contiguous [n_out][B]. */
int sg_maxprod_fwd(const sg_maxprod_plan* plan, const sg_rows* inputs, int64_t B, int32_t clamp01, float* out,
                   int32_t* argmax, sg_stream_t stream);
int sg_maxprod_bwd(const sg_maxprod_plan* plan, const sg_rows* inputs, int64_t B, const int32_t* argmax,
                   sg_rows grad_out, const sg_rows* grad_in, sg_stream_t stream);

/* ---- fused Toeplitz apply chains ---------------------------------------------------
 * v_i = clamp01(v_{i-1} (*) S_i), i = 1..m — a left fold of Toeplitz applies (every Sum-N
 * fold step) as ONE forward and ONE backward launch; per-step arithmetic is the one of
 * sg_damp_apply_fwd/bwd.  All filters have kf rows; v_i has n0 + i (kf - 1) rows.
 * states: sg_chain_states_elems(n0, kf, m, B) floats (a CTA-blocked layout private to the
 * two kernels), written by fwd, read by bwd.  Chains whose longest state exceeds
 * sg_chain_max_rows(kf) rows do not fit in shared memory (cudaErrorNotSupported). */
#define SG_CHAIN_MAX_STEPS 32
typedef struct sg_chain {
  sg_rows base;
  int32_t n0;
  int32_t kf;
  int32_t m;
  int32_t pad_;
  int64_t B;
  sg_rows filters[SG_CHAIN_MAX_STEPS];
  float* states;
} sg_chain;

int64_t sg_chain_states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B);
int32_t sg_chain_max_rows(int32_t kf);
/* rowsum (optional, may be NULL): [B] fp64 sums of each sample's output row, the
 * normaliser loss_nll needs (sg_nll_fwd_rowsum consumes it). */
int sg_chain_fwd(const sg_chain* chain, float* out, double* rowsum, sg_stream_t stream);
int sg_chain_bwd(const sg_chain* chain, const float* grad_out, sg_rows grad_base,
                 const sg_rows* grad_filters, sg_stream_t stream);
/* The same backward when the chain's output feeds loss_nll directly (learn.py:92-119): the
 * upstream gradient rows are generated inside the kernel from the per-sample scalars
 * (target, row sum and picked probability from sg_nll_fwd_rowsum, d loss) exactly as
 * sg_nll_bwd computes them, so the [n_m][B] gradient is never written or read. */
int sg_chain_bwd_nll(const sg_chain* chain, const int64_t* targets, const double* rowsum,
                     const double* picked, const double* grad_loss, sg_rows grad_base,
                     const sg_rows* grad_filters, sg_stream_t stream);

/* 1 when sg_damp_apply_bwd of a short-filter Toeplitz plan (conv == 1) reads its upstream
 * gradient in any layout (the staged kernels); 0: it must be contiguous [n_out][B]. */
int32_t sg_damp_conv_staged(int32_t kf, int32_t n_long, int32_t n_out);

/* ---- fused max-product Toeplitz chain (the north star's max/DAMP variant) ------------
 * The same left fold as sg_chain_* under DampMax (long operand first, kf-row filters):
 * v_i = clamp01(max_s v_{i-1}[s] * S_i[o - s]), first maximal record (s ascending) kept;
 * per step bit-identical to sg_maxprod_fwd/bwd.  states: sg_maxchain_states_elems floats
 * ([rows][B]), argmax: sg_maxchain_argmax_bytes bytes (the argmax tap per step, output,
 * sample); both written by fwd and read by bwd.  rowsum as for sg_chain_fwd. */
int64_t sg_maxchain_states_elems(int32_t n0, int32_t kf, int32_t m, int64_t B);
int64_t sg_maxchain_argmax_bytes(int32_t n0, int32_t kf, int32_t m, int64_t B);
int32_t sg_maxchain_max_rows(int32_t kf);
int sg_maxchain_fwd(const sg_chain* chain, float* out, double* rowsum, uint8_t* argmax, sg_stream_t stream);
int sg_maxchain_bwd(const sg_chain* chain, const uint8_t* argmax, const float* grad_out, sg_rows grad_base,
                    const sg_rows* grad_filters, sg_stream_t stream);

/* ---- fused get_probs -> loss_nll (learn.py:92-119, pass-through clamps) ---------------
 * loss = -(1/B) sum_b log(max(max(p[t_b][b] / (sum_n p[n][b] + 1e-8), 1e-12), 1e-12)),
 * t_b = -1 marks "no mass" (the floor's penalty, no gradient).  fp64 inside.
 * scratch: >= sg_nll_scratch_bytes(n, B) bytes; its first 8 bytes must be zero before the
 * first sg_nll_fwd on it (a self-resetting ticket).  rowsum: [B] doubles, the per-sample
 * sum_n p[n][b] written by the forward for the backward (saved by the caller). */
int64_t sg_nll_scratch_bytes(int64_t n, int64_t B);
int sg_nll_fwd(sg_rows probs, int64_t n, int64_t B, const int64_t* targets, double* loss,
               void* scratch, double* rowsum, sg_stream_t stream);
/* The same loss when the per-sample row sums are already known (rowsum: [B] fp64, e.g.
 * from sg_chain_fwd): one launch that only gathers p[t_b][b]. */
int sg_nll_fwd_rowsum(sg_rows probs, int64_t n, int64_t B, const int64_t* targets,
                      const double* rowsum, double* loss, void* scratch, double* picked,
                      sg_stream_t stream);  /* picked (optional): [B] p[t_b][b] as fp64 */
/* grad[n][b] = -(g/B) / c_b * (delta(n, t_b) / (s_b + 1e-8) - p[t_b][b] / (s_b + 1e-8)^2) */
int sg_nll_bwd(sg_rows probs, int64_t n, int64_t B, const int64_t* targets,
               const double* grad_loss, const double* rowsum, sg_rows grad, sg_stream_t stream);

/* ---- row gather (filter / placement / inverse scatter), any tag kind -----------------
 * dst row r = src row idx[r] (idx -1 -> zero row); rows are row_bytes contiguous bytes. */
int sg_rows_gather(const void* src, const int32_t* idx, int64_t n_rows, int64_t row_bytes,
                   void* dst, sg_stream_t stream);

/* ---- DTKP-AM (top-k proofs) --------------------------------------------------------- */
typedef struct sg_dtkp_operand {
  const uint64_t* member; /* [rows][K][W][B] */
  const uint8_t* present; /* [rows][K][B]    */
  int32_t rows;
  int32_t W;              /* words stored for this operand (<= W_out; missing words are 0) */
} sg_dtkp_operand;

typedef struct sg_dtkp_apply_desc {
  int32_t arity;          /* number of conjoined inputs (1 = group_disj / union / merge)    */
  int32_t K;              /* proofs kept per tag                                            */
  int32_t W;              /* output words = ceil(I / 64)                                    */
  int32_t I;              /* registry width (columns of p)                                  */
  int64_t B;
  sg_dtkp_operand ops[SG_MAX_ARITY];
  sg_dtkp_operand op_tail;  /* arity == 1 only: record r >= ops[0].rows reads op_tail row r - ops[0].rows */
  const float* p;          /* registry probabilities [I][B] (fp32; ranking keys are fp64 of these) */
  sg_segsum seg;           /* segments = output symbols; records = input positions           */
  uint64_t* out_member;    /* [seg.n_seg][K][W][B] */
  uint8_t* out_present;    /* [seg.n_seg][K][B]    */
  uint64_t* scratch_member;/* [seg.n_partial][K][W][B] partial top-k of split segments      */
  uint8_t* scratch_present;/* [seg.n_partial][K][B] */
  sg_segsum merge;         /* arity-1 merge of partial rows (seg.n_split segments)           */
  int32_t* sched;          /* optional work counters, ceil(B/32) + 1 int32, zero before the
                            * first use and left zero by every launch (the last CTA resets
                            * them): warps then take items dynamically instead of by the
                            * static seg.blk partition.  Launches that may run concurrently
                            * need distinct buffers.  NULL = static partition.            */
  /* Two-level merge: when merge.n_split > 0, merge items that are themselves split write
   * their partial lists to scratch2 (merge.n_partial rows) and merge2 (merge.n_split
   * segments, records = scratch2 rows) combines them into the output.  Every level keeps
   * the record order, so the result equals a single serial merge bit for bit.          */
  sg_segsum merge2;
  uint64_t* scratch2_member; /* [merge.n_partial][K][W][B] */
  uint8_t* scratch2_present; /* [merge.n_partial][K][B]    */
  /* Fused conj -> group_disj (arity == 1 only; inner_arity == 0 disables it).  The single
   * operand of this apply is the output of a binary (arity-2) apply that is never
   * materialised — HWF's final eval over the 208767 formulas of its last concat step
   * (programs.py:117-145).  seg.recs then holds the BINARY apply's records (rec_words >= 2:
   * row of inner_ops[0], row of inner_ops[1]) in this apply's segment order: for every
   * record of this apply (an intermediate symbol) the conj records of that symbol in their
   * ordinal order, the last one marked by bit 31 of its second word.  Each symbol's tag is
   * built exactly as the binary apply builds its output row (per-record normalised conj,
   * provenance.py:328-341, streamed through a top-k, :352-364) and its rows stream into this
   * apply's top-k in rank order — bit-identical to the two launches, while the intermediate
   * tag never touches HBM.  ops[0] and op_tail are not read.                            */
  int32_t inner_arity;
  /* seg_packed != 0: seg's items (.x = first segment, .w = -1) may hold runs of WHOLE
   * segments; word 0 of a segment's last record carries bit 31 (rows are < 2^31).  Items
   * with .w >= 0 are pieces of one split segment, as always.  The merges are never packed. */
  int32_t seg_packed;
  sg_dtkp_operand inner_ops[2];
  /* rows_ranked != 0: every operand tag holds its present rows first in non-increasing key
   * order (true for every normalised tag: kernel outputs, input tags, row gathers).  A
   * streaming (arity-1) apply then stops reading a tag at its first row that cannot enter
   * the full top-k — its later rows rank no higher, and a tie loses to the earlier row.
   * 0 (e.g. hand-built tags): every row is ranked.                                      */
  int32_t rows_ranked;
  int32_t rows_ranked_pad_;
} sg_dtkp_apply_desc;

int sg_dtkp_apply(const sg_dtkp_apply_desc* d, sg_stream_t stream);

/* P[n][b] = clamp01( sum_r present * prod_{j in row r} p[j][b] )  (fp64 inside, fp32 out) */
int sg_dtkp_probs_fwd(const uint64_t* member, const uint8_t* present, int32_t N, int32_t K,
                      int32_t W, const float* p, int32_t I, int64_t B, float* out,
                      sg_stream_t stream);
/* dp[j][b] = sum_{n,r: j in row} g[n][b] * present * prod_{j' != j} p[j'][b] (exact zeros rule).
 * scratch: >= sg_dtkp_probs_bwd_scratch(N, I, B) bytes. */
int64_t sg_dtkp_probs_bwd_scratch(int32_t N, int32_t I, int64_t B);
int sg_dtkp_probs_bwd(const uint64_t* member, const uint8_t* present, int32_t N, int32_t K,
                      int32_t W, const float* p, int32_t I, int64_t B, const float* grad_out,
                      float* grad_p, void* scratch, sg_stream_t stream);

/* Drop-in for _dtkpcore.dedup_topk (device buffers, caller-allocated outputs):
 *   member u8 [M][R][I], present u8 [M][R], p f64 [M][I]  ->
 *   out_member u8 [M][k][I], out_present u8 [M][k]
 * Dedup identical present rows (first wins), rank by fp64 product of p over member
 * columns in ascending column order, ties by row index, copy source bytes. */
int sg_dedup_topk(const uint8_t* member, const uint8_t* present, const double* p, int64_t M,
                  int32_t R, int32_t I, int32_t k, uint8_t* out_member, uint8_t* out_present,
                  sg_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SGB200_H */
