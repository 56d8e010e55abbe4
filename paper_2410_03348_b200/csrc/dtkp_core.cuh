// DTKP-AM device core: the streaming top-k set, ranking keys and the fused apply kernel.
// See dtkp.cu for the semantics; this header is instantiated once per K (dtkp_apply_k.cu)
// so the eight K variants compile in parallel.
#pragma once
#include <algorithm>
#include "common.cuh"

#ifndef SG_DTKP_WAVES  // resident waves of apply CTAs per launch (each strides over work blocks)
#define SG_DTKP_WAVES 3
#endif
#ifndef SG_DTKP_MINB  // > 0 overrides the per-variant register policy (dtkp_min_blocks)
#define SG_DTKP_MINB 0
#endif
#ifndef SG_DTKP_CONJ_PREFETCH_MAXK  // conj kernels prefetch the next record for K <= this
#define SG_DTKP_CONJ_PREFETCH_MAXK 2
#endif
#ifndef SG_DTKP_STREAM_PREFETCH  // streaming (arity-1) kernel loads the next record ahead
#define SG_DTKP_STREAM_PREFETCH 0
#endif
#ifndef SG_DTKP_FUSED_MINB  // resident CTAs/SM asked of the fused conj -> group_disj (K <= 3)
#define SG_DTKP_FUSED_MINB 5
#endif
#ifndef SG_DTKP_CONJ3_MINB  // resident CTAs/SM asked of the binary conj at K = 3
#define SG_DTKP_CONJ3_MINB 6
#endif
#ifndef SG_DTKP_UNROLL_K
#define SG_DTKP_UNROLL_K 4
#endif

namespace sg {

// Running top-k of distinct proofs ordered by (key desc, stream position asc).
template <int K, int WT>
struct TopK {
  uint64_t m[K][WT];
  double key[K];
  int idx[K];
  int n;

  __device__ __forceinline__ void clear() { n = 0; }

  // Insert a candidate that comes after every previously streamed candidate
  // (_dtkpcore.pyx:58-94 semantics: first occurrence wins, ties keep stream order).
  __device__ __forceinline__ void insert(const uint64_t (&mm)[WT], double kk, int id) {
    if (n == K && !(kk > key[K - 1])) return;
    bool dup = false;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      bool eq = i < n;
#pragma unroll
      for (int w = 0; w < WT; ++w) eq = eq && (m[i][w] == mm[w]);
      dup = dup || eq;
    }
    if (dup) return;
    int pos = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) pos += (i < n && key[i] >= kk) ? 1 : 0;
#pragma unroll
    for (int i = K - 1; i >= 1; --i) {
      if (i > pos) {
#pragma unroll
        for (int w = 0; w < WT; ++w) m[i][w] = m[i - 1][w];
        key[i] = key[i - 1];
        idx[i] = idx[i - 1];
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i == pos) {
#pragma unroll
        for (int w = 0; w < WT; ++w) m[i][w] = mm[w];
        key[i] = kk;
        idx[i] = id;
      }
    }
    n = n < K ? n + 1 : K;
  }

  // Copy entry q (runtime index) out of the register arrays without local memory.
  __device__ __forceinline__ void get(int q, uint64_t (&mm)[WT], double& kk) const {
#pragma unroll
    for (int w = 0; w < WT; ++w) mm[w] = 0ull;
    kk = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i == q) {
#pragma unroll
        for (int w = 0; w < WT; ++w) mm[w] = m[i][w];
        kk = key[i];
      }
    }
  }
};

// One sample's probability column staged in shared memory: fp64 [I][32] when it fits,
// else fp32 [I][32] upcast on read (identical keys: the registry values are fp32).
struct PCol {
  const double* smd;
  const float* smf;
  bool dbl;
  int one;  // index of a staged column holding exactly 1.0 (= I): the filler of proof_key
  __device__ __forceinline__ double operator()(int j) const {
    return dbl ? smd[(size_t)j * kWarp] : (double)smf[(size_t)j * kWarp];
  }
};

static constexpr size_t kMaxPTile = 192 * 1024;

// Staging mode for a registry of I columns (+ the 1.0 column): 2 = fp64, 1 = fp32, 0 =
// does not fit.
__host__ __device__ inline int ptile_mode(int I) {
  if ((size_t)(I + 1) * kWarp * sizeof(double) <= kMaxPTile) return 2;
  if ((size_t)(I + 1) * kWarp * sizeof(float) <= kMaxPTile) return 1;
  return 0;
}

__host__ __device__ inline size_t ptile_bytes(int I) {
  return (size_t)(I + 1) * kWarp * (ptile_mode(I) == 2 ? sizeof(double) : sizeof(float));
}

__device__ __forceinline__ PCol stage_pcol(void* tile, const float* __restrict__ p, int I, int64_t B, int64_t b,
                                           int lane, int warp, int nwarps) {
  const bool dbl = ptile_mode(I) == 2;
  // eight independent loads in flight per thread (a serial load -> store loop here was
  // ~40% of a short DTKP launch: one L2 round trip per column)
  constexpr int U = 8;
  for (int j0 = warp; j0 < I; j0 += U * nwarps) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * nwarps;
      v[u] = j < I ? __ldg(p + (size_t)j * B + b) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * nwarps;
      if (j < I) {
        if (dbl)
          reinterpret_cast<double*>(tile)[(size_t)j * kWarp + lane] = (double)v[u];
        else
          reinterpret_cast<float*>(tile)[(size_t)j * kWarp + lane] = v[u];
      }
    }
  }
  if (warp == 0) {  // column I = 1.0 exactly
    if (dbl)
      reinterpret_cast<double*>(tile)[(size_t)I * kWarp + lane] = 1.0;
    else
      reinterpret_cast<float*>(tile)[(size_t)I * kWarp + lane] = 1.f;
  }
  return PCol{reinterpret_cast<const double*>(tile) + lane, reinterpret_cast<const float*>(tile) + lane, dbl, I};
}

// fp64 product of member probabilities in ascending column order (_dtkpcore.pyx:53-57).
// Set bits are consumed four at a time: the four shared-memory loads are issued together
// and the products are taken in ascending order; missing slots multiply by 1.0, which is
// exact in IEEE arithmetic, so the result is bit-identical to the one-bit-at-a-time loop.
// `start` continues a product: proof_key(b, pc, proof_key(a, pc)) == proof_key(a | b, pc)
// bit for bit when every member of a precedes every member of b (the fold is the same
// sequence of multiplies).
#ifndef SG_DTKP_KEY32  // 0: the 64-bit scan with selected fillers (A/B tests)
#define SG_DTKP_KEY32 1
#endif
template <int WT>
__device__ __forceinline__ double proof_key(const uint64_t (&mm)[WT], const PCol& pc, double start = 1.0) {
  double prod = start;
#if SG_DTKP_KEY32
  // 32-bit halves (one FLO per bit instead of a 64-bit find-first-set), and a group's
  // missing slots read the staged 1.0 column instead of selecting 1.0 after the load.
  // (A member-count switch to 64-bit words for sparse proofs measured slower on both
  // HWF-7 and CLUTRR: the branch and its registers cost more than the part-filled groups.)
#pragma unroll
  for (int h = 0; h < 2 * WT; ++h) {
    uint32_t x = (h & 1) ? (uint32_t)(mm[h >> 1] >> 32) : (uint32_t)mm[h >> 1];
    while (x) {
      int j[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        j[u] = x ? h * 32 + __ffs((int)x) - 1 : pc.one;
        x &= x - 1;
      }
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = pc(j[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) prod *= v[u];
    }
  }
  return prod;
#else
#pragma unroll
  for (int w = 0; w < WT; ++w) {
    uint64_t x = mm[w];
    while (x) {
      int j[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ok[u] = x != 0;
        j[u] = ok[u] ? (w * 64 + __ffsll((long long)x) - 1) : 0;
        x &= x - 1;
      }
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = pc(j[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) prod *= ok[u] ? v[u] : 1.0;
    }
  }
  return prod;
#endif
}

struct DtkpK {
  sg_dtkp_operand ops[SG_MAX_ARITY];
  sg_dtkp_operand tail;
  int32_t arity, K, W, I;
  int64_t B;
  const float* p;
  const int32_t* recs;
  int32_t rec_words;
  const int32_t* items;
  const int32_t* blk;
  int32_t n_blk;  // work blocks; CTAs stride over them (set by the launcher)
  int32_t n_items;
  int32_t* sched;  // optional [gx + 1] zeroed counters: dynamic item schedule
  uint64_t* out_m;
  uint8_t* out_p;
  uint64_t* scr_m;
  uint8_t* scr_p;
  // fused conj -> group_disj (AR == 3): the binary conj's operands (records in recs)
  sg_dtkp_operand inner[2];
  int32_t fused;
  int32_t packed;  // items may hold runs of whole segments (record word 0 bit 31 = segment end)
  int32_t ranked;  // operand rows are in non-increasing key order (streaming may stop early)
};

template <int WT>
__device__ __forceinline__ void load_row(const sg_dtkp_operand& op, int K, int64_t B, int64_t b, int r, int q,
                                         uint64_t (&mm)[WT]) {
  const unsigned long long* base =
      reinterpret_cast<const unsigned long long*>(op.member) + ((size_t)r * K + q) * (size_t)op.W * B + b;
#pragma unroll
  for (int w = 0; w < WT; ++w) mm[w] = (w < op.W) ? __ldg(base + (size_t)w * B) : 0ull;
}

__device__ __forceinline__ bool row_present(const sg_dtkp_operand& op, int K, int64_t B, int64_t b, int r, int q) {
  return __ldg(op.present + ((size_t)r * K + q) * B + b) != 0;
}

// All K proof rows of one tag (one symbol, one sample) in registers, loaded with
// K * (WT + 1) independent loads and no data-dependent branch (memory-level parallelism).
template <int K, int WT>
struct TagRows {
  uint64_t m[K][WT];
  uint32_t pres;  // bit q = row q present

  __device__ __forceinline__ void load(const sg_dtkp_operand& op, int64_t B, int64_t b, int r) {
    const uint8_t* pp = op.present + (size_t)r * K * B + b;
    const unsigned long long* base =
        reinterpret_cast<const unsigned long long*>(op.member) + (size_t)r * K * (size_t)op.W * B + b;
    uint32_t p = 0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      p |= (__ldg(pp + (size_t)q * B) != 0 ? 1u : 0u) << q;
#pragma unroll
      for (int w = 0; w < WT; ++w) m[q][w] = (w < op.W) ? __ldg(base + ((size_t)q * op.W + w) * B) : 0ull;
    }
    pres = p;
  }

  // Row q (runtime index) without local memory: unrolled select.
  __device__ __forceinline__ void row(int q, uint64_t (&mm)[WT]) const {
#pragma unroll
    for (int w = 0; w < WT; ++w) mm[w] = m[0][w];
#pragma unroll
    for (int i = 1; i < K; ++i) {
      if (i == q) {
#pragma unroll
        for (int w = 0; w < WT; ++w) mm[w] = m[i][w];
      }
    }
  }
};

__device__ __forceinline__ int rec_row(const DtkpK& a, int c, int i) { return __ldg(a.recs + (size_t)c * a.rec_words + i); }

// Stream the candidates of conj(A, Bt) — all present row pairs OR-ed, in candidate order
// ra*kb + rb (provenance.py:328-341) — into the running top-k T.  With T cleared first
// this is the conj's own normalisation (_normalize :366-379).  Streaming them straight into
// the group_disj's running top-k (provenance.py:352-364) instead of normalising each combo
// first gives the SAME rows in the same order: a candidate in the top-k of the whole
// segment has fewer than k better candidates in its own combo, so it survives that combo's
// normalisation; normalisation keeps the candidate order among equal keys, dedup keeps the
// first occurrence either way, and the top-k of a union equals the top-k of the union of
// the members' top-k lists (SURVEY §7 hard part 2).  Only n-ary folds (arity >= 3) must
// normalise between steps: there the truncation feeds the next OR.
template <int K, int WT>
__device__ __forceinline__ void conj_into(TopK<K, WT>& T, const TagRows<K, WT>& A, const TagRows<K, WT>& Bt,
                                          const PCol& pc) {
  constexpr int kUnrollK = K <= SG_DTKP_UNROLL_K ? K : 1;
#pragma unroll (kUnrollK)
  for (int qa = 0; qa < K; ++qa) {
    if (!((A.pres >> qa) & 1u)) continue;
    uint64_t ma[WT];
    A.row(qa, ma);
#pragma unroll (kUnrollK)
    for (int qb = 0; qb < K; ++qb) {
      if (!((Bt.pres >> qb) & 1u)) continue;
      uint64_t mm[WT];
      Bt.row(qb, mm);
#pragma unroll
      for (int w = 0; w < WT; ++w) mm[w] |= ma[w];
      T.insert(mm, proof_key<WT>(mm, pc), 0);
    }
  }
}

// Highest / lowest member column of a proof row (-1 / INT_MAX when it has none).
template <int WT>
__device__ __forceinline__ int hi_col(const uint64_t (&m)[WT]) {
  int h = -1;
#pragma unroll
  for (int w = 0; w < WT; ++w)
    if (m[w]) h = w * 64 + 63 - __clzll((long long)m[w]);
  return h;
}
template <int WT>
__device__ __forceinline__ int lo_col(const uint64_t (&m)[WT]) {
  int l = 0x7fffffff;
#pragma unroll
  for (int w = WT - 1; w >= 0; --w)
    if (m[w]) l = w * 64 + __ffsll((long long)m[w]) - 1;
  return l;
}
template <int WT>
__device__ __forceinline__ bool one_member(const uint64_t (&m)[WT]) {
  int c = 0;
#pragma unroll
  for (int w = 0; w < WT; ++w) c += __popcll(m[w]);
  return c == 1;
}

#ifndef SG_DTKP_KEY_CONT  // 0: every conj candidate's key is a full product (A/B tests)
#define SG_DTKP_KEY_CONT 1
#endif
#ifndef SG_DTKP_KEYED_MAXK  // largest K whose binary conj keeps left-row keys (registers)
#define SG_DTKP_KEYED_MAXK 3
#endif
#ifndef SG_DTKP_CONJ5_MINB  // resident CTAs/SM asked of the binary conj at 3 < K <= 5
#define SG_DTKP_CONJ5_MINB 4
#endif
#ifndef SG_DTKP_STREAM5_MINB  // resident CTAs/SM asked of the streaming kernel at 3 < K <= 5
#define SG_DTKP_STREAM5_MINB 5
#endif
#ifndef SG_DTKP_FIRST_FILL  // 0: the first record of a segment is inserted candidate by candidate
#define SG_DTKP_FIRST_FILL 1
#endif
#ifndef SG_DTKP_PRUNE  // 0: no upper-bound pruning of binary conj candidates (A/B tests)
#define SG_DTKP_PRUNE 1
#endif

// Keys of the K rows of a left conj operand (0 for absent rows), computed once per loaded
// tag and reused by every record of an item that conjoins the same left row.
template <int K>
struct RowKeys {
  double k[K];
  __device__ __forceinline__ double at(int q) const {
    double v = k[0];
#pragma unroll
    for (int i = 1; i < K; ++i)
      if (i == q) v = k[i];
    return v;
  }
  template <int WT>
  __device__ __forceinline__ void compute(const TagRows<K, WT>& A, const PCol& pc) {
#pragma unroll
    for (int q = 0; q < K; ++q) k[q] = ((A.pres >> q) & 1u) ? proof_key<WT>(A.m[q], pc) : 0.0;
  }
};

// Binary conj streamed into the segment's top-k S (AR = 2, K <= 3) with the left rows'
// keys known (AK).  Same candidate order and the same inserts as conj_into; two exact
// shortcuts:
//  * bound: with every registry probability of the sample in [0, 1] (le1), the ascending
//    fp64 product over a union never exceeds the product over its left part (each extra
//    factor is <= 1 and rounding is monotone), so once S is full a left row whose key is
//    not above S's k-th key contributes nothing — insert() would reject each of its
//    candidates after computing their keys; the row is skipped before;
//  * continuation: when every member of the right row follows the left row's, the
//    union's product is the left key continued over the right row (one multiply for a
//    single-member row), the same multiplies in the same order as proof_key.
template <int K, int WT>
__device__ __forceinline__ void conj_keyed(TopK<K, WT>& S, const TagRows<K, WT>& A, const RowKeys<K>& AK,
                                           const TagRows<K, WT>& Bt, bool le1, bool ranked, const PCol& pc) {
  constexpr int kUnrollK = K <= SG_DTKP_UNROLL_K ? K : 1;
  if (SG_DTKP_FIRST_FILL && ranked && S.n == 0 && Bt.pres == 1u && (A.pres & (A.pres + 1u)) == 0u) {
    // First record of a segment, one single-member right row that follows every left row:
    // the candidates a_q | b are distinct (the a_q are) and their keys key(a_q) * p_b are
    // non-increasing in q (a ranked tag, one non-negative factor), so the inserts would
    // append them in order — S takes them directly.
    uint64_t mb[WT];
    Bt.row(0, mb);
    const int lb = lo_col<WT>(mb);
    bool ok = one_member<WT>(mb);
#pragma unroll
    for (int q = 0; q < K; ++q)
      if ((A.pres >> q) & 1u) ok = ok && hi_col<WT>(A.m[q]) < lb;
    if (ok) {
      const double pb = pc(lb);
      int n = 0;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if ((A.pres >> q) & 1u) {
#pragma unroll
          for (int w = 0; w < WT; ++w) S.m[q][w] = A.m[q][w] | mb[w];
          S.key[q] = AK.k[q] * pb;
          S.idx[q] = 0;
          ++n;
        }
      }
      S.n = n;
      return;
    }
  }
#pragma unroll (kUnrollK)
  for (int qa = 0; qa < K; ++qa) {
    if (!((A.pres >> qa) & 1u)) continue;
    const double ka = AK.at(qa);
    if (SG_DTKP_PRUNE && le1 && S.n == K && !(ka > S.key[K - 1])) continue;
    uint64_t ma[WT];
    A.row(qa, ma);
    const int ha = hi_col<WT>(ma);
#pragma unroll (kUnrollK)
    for (int qb = 0; qb < K; ++qb) {
      if (!((Bt.pres >> qb) & 1u)) continue;
      uint64_t mb[WT], mm[WT];
      Bt.row(qb, mb);
#pragma unroll
      for (int w = 0; w < WT; ++w) mm[w] = mb[w] | ma[w];
      double kk;
      const int lb = lo_col<WT>(mb);
      if (SG_DTKP_KEY_CONT && ha < lb)
        kk = one_member<WT>(mb) ? ka * pc(lb) : proof_key<WT>(mb, pc, ka);
      else
        kk = proof_key<WT>(mm, pc);
      S.insert(mm, kk, 0);
    }
  }
}

// Stream the retained rows of T (rank order) into S: the group_disj of a column of tags
// (same mask, same p -> same key as a recomputation, so the key is reused).
template <int K, int WT>
__device__ __forceinline__ void stream_rows(TopK<K, WT>& S, const TopK<K, WT>& T) {
  constexpr int kUnrollK = K <= SG_DTKP_UNROLL_K ? K : 1;
#pragma unroll (kUnrollK)
  for (int q = 0; q < K; ++q) {
    if (q >= T.n) break;
    uint64_t mm[WT];
    double kk;
    T.get(q, mm, kk);
    // T is ranked: once a row cannot enter a full S, none of the later ones can
    if (S.n == K && !(kk > S.key[K - 1])) break;
    S.insert(mm, kk, 0);
  }
}

// Write the retained rows of S as tag row `row` of (om, opr) for this lane's sample.
template <int K, int WT>
__device__ __forceinline__ void emit_rows(const DtkpK& a, const TopK<K, WT>& S, uint64_t* om_base, uint8_t* op_base,
                                          int row, int64_t b0) {
  uint64_t* om = om_base + (size_t)row * K * a.W * a.B;
  uint8_t* opr = op_base + (size_t)row * K * a.B;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const bool live = q < S.n;
    opr[(size_t)q * a.B + b0] = live ? 1 : 0;
#pragma unroll
    for (int w = 0; w < WT; ++w)
      if (w < a.W) om[((size_t)q * a.W + w) * a.B + b0] = live ? S.m[q][w] : 0ull;
  }
}

constexpr int kRowMask = 0x7fffffff;  // record word 0 bit 31: last record of a segment (packed items)

// One work item for one sample: stream its records through the top-k set and write the
// retained rows.  An item is a piece of one (long, split) segment written to scratch
// (item.w >= 0), one whole segment (item.w < 0), or — in a packed problem (a.packed) —
// a run of WHOLE short segments starting at segment item.x: each record whose word 0
// carries bit 31 closes the current segment (its rows are written, the set is cleared and
// the next segment begins).  Packing turns e.g. HWF-7 step 7 (208,767 segments of ~1.5
// records) into items of ~48 records, so the per-item chain (work counter atomic ->
// item -> records) is paid once per 30 segments instead of once per segment.
// AR: 1 = union / group_disj streaming, 2 = binary conj fold, 0 = conj fold of >= 3
// operands, 3 = the fused conj -> group_disj (sg_dtkp_apply_desc.inner_arity): records are
// binary-conj records (rows of inner[0], inner[1]) grouped by intermediate symbol, the last
// record of each intermediate flagged by bit 31 of its second word.  Each is its own kernel,
// so the streaming kernel does not carry the conj fold's registers (occupancy) or code.
template <int K, int WT, int AR>
__device__ __forceinline__ void apply_item(const DtkpK& a, int it, int64_t b, int64_t b0, bool bval, const PCol& pc,
                                           bool le1) {
  constexpr int kUnrollK = K <= SG_DTKP_UNROLL_K ? K : 1;
  const int4 item = __ldg(reinterpret_cast<const int4*>(a.items) + it);
  const bool multi = a.packed && item.w < 0;  // segments close at flagged records
  int seg = item.x;
  TopK<K, WT> S;
  S.clear();
  auto close_seg = [&](int word0) {
    if (multi && word0 < 0) {
      if (bval) emit_rows<K, WT>(a, S, a.out_m, a.out_p, seg, b0);
      S.clear();
      ++seg;
    }
  };
  if constexpr (AR == 1) {
    // group_disj / union / merge: stream the stored rows of every record, in order;
    // the next record's rows are loaded after the current one is ranked
    TagRows<K, WT> cur;
    auto fetch = [&](int r) {
      r &= kRowMask;
      if (r >= a.ops[0].rows)
        cur.load(a.tail, a.B, b, r - a.ops[0].rows);
      else
        cur.load(a.ops[0], a.B, b, r);
    };
    int w0 = item.y < item.z ? rec_row(a, item.y, 0) : 0;
    if (item.y < item.z) fetch(w0);
    for (int c = item.y; c < item.z; ++c) {
      const int wn = c + 1 < item.z ? rec_row(a, c + 1, 0) : 0;
#pragma unroll (kUnrollK)
      for (int q = 0; q < K; ++q) {
        if (!((cur.pres >> q) & 1u)) continue;
        uint64_t mm[WT];
        cur.row(q, mm);
        const double kk = proof_key<WT>(mm, pc);
        // a ranked tag's later rows cannot enter a full top-k this row cannot enter
        if (a.ranked && S.n == K && !(kk > S.key[K - 1])) break;
        S.insert(mm, kk, 0);
      }
      close_seg(w0);
      if (c + 1 < item.z) fetch(wn);
      w0 = wn;
    }
  } else if constexpr (AR == 3) {
    // fused conj -> group_disj: M collects an intermediate symbol's tag (the top-k over its
    // conj records, what an arity-2 apply writes as its row); at the symbol's last record
    // M's rows stream into S in rank order, as the group_disj of the materialised tag reads
    const sg_dtkp_operand& o0 = a.inner[0];
    const sg_dtkp_operand& o1 = a.inner[1];
    TagRows<K, WT> A, Bt;
    int ra = 0, rbf = 0, ran = 0, rbn = 0;
    if (item.y < item.z) {
      ra = rec_row(a, item.y, 0);
      rbf = rec_row(a, item.y, 1);
      A.load(o0, a.B, b, ra & kRowMask);
      Bt.load(o1, a.B, b, rbf & kRowMask);
    }
    if (item.y + 1 < item.z) {
      ran = rec_row(a, item.y + 1, 0);
      rbn = rec_row(a, item.y + 1, 1);
    }
    TopK<K, WT> M;
    M.clear();
    for (int c = item.y; c < item.z; ++c) {
      const bool more = c + 1 < item.z;
      const int rna = ran, rnb = rbn;
      if (c + 2 < item.z) {
        ran = rec_row(a, c + 2, 0);
        rbn = rec_row(a, c + 2, 1);
      }
      conj_into<K, WT>(M, A, Bt, pc);
      if (rbf < 0) {  // last conj record of this intermediate symbol
        stream_rows<K, WT>(S, M);
        M.clear();
      }
      close_seg(ra);
      if (more) {
        ra = rna;
        rbf = rnb;
        A.load(o0, a.B, b, rna & kRowMask);
        Bt.load(o1, a.B, b, rnb & kRowMask);
      }
    }
  } else {
    // conj fold, normalised after every step (candidate order ra*kb + rb)
    TagRows<K, WT> A, Bt, An, Bn;
    int wa = 0, ran = 0, rbn = 0;
    if (item.y < item.z) {
      wa = rec_row(a, item.y, 0);
      A.load(a.ops[0], a.B, b, wa & kRowMask);
      Bt.load(a.ops[1], a.B, b, rec_row(a, item.y, 1));
    }
    if (item.y + 1 < item.z) {
      ran = rec_row(a, item.y + 1, 0);
      rbn = rec_row(a, item.y + 1, 1);
    }
    // next record's rows held in registers only while K is small (their registers cost
    // occupancy); otherwise loaded after the current record
    constexpr bool kPf = K <= SG_DTKP_CONJ_PREFETCH_MAXK;
    // AR 2, K <= 3: the left rows' keys stay valid while consecutive records conjoin the
    // same left row (records are grouped by output symbol, and e.g. a prefix extended by
    // every symbol of the next input is a run of records with one left row).  At K = 5 the
    // key registers spill and CLUTRR-style closures lost 9-15%, so larger K stream plainly.
    constexpr bool kKeyed = AR == 2 && K <= SG_DTKP_KEYED_MAXK;
    RowKeys<K> AK;
    bool ak_ok = false;
    for (int c = item.y; c < item.z; ++c) {
      const bool more = c + 1 < item.z;
      const int rna = ran, rnb = rbn;
      const bool same_a = kKeyed && (rna & kRowMask) == (wa & kRowMask);
      if (kPf && more) {
        if (!same_a) An.load(a.ops[0], a.B, b, rna & kRowMask);
        Bn.load(a.ops[1], a.B, b, rnb);
      }
      if (c + 2 < item.z) {
        ran = rec_row(a, c + 2, 0);
        rbn = rec_row(a, c + 2, 1);
      }
      if constexpr (AR == 2) {
        // exact: see conj_into / conj_keyed
        if constexpr (kKeyed) {
          if (!ak_ok) {
            AK.compute<WT>(A, pc);
            ak_ok = true;
          }
          conj_keyed<K, WT>(S, A, AK, Bt, le1, a.ranked != 0, pc);
        } else {
          conj_into<K, WT>(S, A, Bt, pc);
        }
      } else {
        TopK<K, WT> T;
        T.clear();
        conj_into<K, WT>(T, A, Bt, pc);
#pragma unroll 1
        for (int i = 2; i < a.arity; ++i) {
          TagRows<K, WT> Ci;
          Ci.load(a.ops[i], a.B, b, rec_row(a, c, i));
          TopK<K, WT> U;
          U.clear();
#pragma unroll (kUnrollK)
          for (int qa = 0; qa < K; ++qa) {
            if (qa >= T.n) break;
            uint64_t ma[WT];
            double ka;
            T.get(qa, ma, ka);
#pragma unroll (kUnrollK)
            for (int qb = 0; qb < K; ++qb) {
              if (!((Ci.pres >> qb) & 1u)) continue;
              uint64_t mm[WT];
              Ci.row(qb, mm);
#pragma unroll
              for (int w = 0; w < WT; ++w) mm[w] |= ma[w];
              U.insert(mm, proof_key<WT>(mm, pc), 0);
            }
          }
          T = U;
        }
        stream_rows<K, WT>(S, T);
      }
      close_seg(wa);
      if (more) {
        wa = rna;
        if constexpr (kPf) {
          if (!same_a) A = An;
          Bt = Bn;
        } else {
          if (!same_a) A.load(a.ops[0], a.B, b, rna & kRowMask);
          Bt.load(a.ops[1], a.B, b, rnb);
        }
        if (!same_a) ak_ok = false;
      }
    }
  }
  if (bval && (!multi || item.y == item.z)) {  // (a packed item without records = one empty segment)
    if (item.w < 0)
      emit_rows<K, WT>(a, S, a.out_m, a.out_p, item.x, b0);
    else
      emit_rows<K, WT>(a, S, a.scr_m, a.scr_p, item.w, b0);
  }
}

// Resident CTAs per SM the register allocator is asked for: the highest that compiles
// without spills at K <= 3 / K <= 5 and W <= 2 (ptxas -v), else whatever the kernel needs.
__host__ __device__ constexpr int dtkp_min_blocks(int K, int WT, int AR) {
  // binary conj (AR 2) streams its candidates straight into the segment's top-k (no
  // per-combo top-k set): 6 / 4 CTAs per SM at K <= 3 / K <= 5 without spills
  return SG_DTKP_MINB > 0 ? SG_DTKP_MINB
         : (WT <= 2 && K <= 3) ? (AR == 1 ? (SG_DTKP_STREAM_PREFETCH ? 5 : 6)
                                  : AR == 2 ? (K > SG_DTKP_CONJ_PREFETCH_MAXK ? SG_DTKP_CONJ3_MINB : 4)
                                  : AR == 3 ? SG_DTKP_FUSED_MINB : 1)
         : (WT <= 2 && K <= 5 && AR == 1) ? SG_DTKP_STREAM5_MINB
         : (WT <= 2 && K <= 5 && AR == 2 && K > SG_DTKP_CONJ_PREFETCH_MAXK) ? SG_DTKP_CONJ5_MINB
         : 1;
}

template <int K, int WT, int AR>
__global__ void __launch_bounds__(128, dtkp_min_blocks(K, WT, AR)) k_dtkp_apply(const DtkpK a) {
  extern __shared__ __align__(16) unsigned char ptile_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kWarp + lane;
  const bool bval = b0 < a.B;
  const int64_t b = bval ? b0 : a.B - 1;
  const PCol pc = stage_pcol(ptile_raw, a.p, a.I, a.B, b, lane, warp, nwarps);
  __syncthreads();
  // binary conj: whether every registry probability of this sample lies in [0, 1] (the
  // bound of conj_keyed)
  bool le1 = true;
  if (AR == 2 && K <= SG_DTKP_KEYED_MAXK) {
    for (int j = 0; j < a.I; ++j) {
      const double v = pc(j);
      le1 = le1 && v >= 0.0 && v <= 1.0;
    }
  }

  if (a.sched != nullptr) {
    // dynamic: every warp takes the next item of its 32-sample column from a counter, so
    // the CTAs of one resident wave stay busy until the column's items run out
    int* ctr = a.sched + blockIdx.x;
    for (;;) {
      int it = 0;
      if (lane == 0) it = atomicAdd(ctr, 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= a.n_items) break;
      apply_item<K, WT, AR>(a, it, b, b0, bval, pc, le1);
    }
    // the last CTA out re-zeroes the counters for the next launch that uses the buffer
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned total = gridDim.x * gridDim.y;
      if (atomicAdd(reinterpret_cast<unsigned*>(a.sched + gridDim.x), 1u) == total - 1) {
        for (unsigned x = 0; x < gridDim.x; ++x) a.sched[x] = 0;
        a.sched[gridDim.x] = 0;
      }
    }
    return;
  }
  // static: CTAs stride over the work blocks; the probability tile is staged once per CTA
  for (int bk = blockIdx.y; bk < a.n_blk; bk += gridDim.y) {
    const int it0 = __ldg(a.blk + bk), it1 = __ldg(a.blk + bk + 1);
    for (int it = it0 + warp; it < it1; it += nwarps) apply_item<K, WT, AR>(a, it, b, b0, bval, pc, le1);
  }
}

template <int K, int WT, int AR>
static int launch_apply_kwa(const DtkpK& k, int n_blocks, cudaStream_t st) {
  const int mode = ptile_mode(k.I);
  if (mode == 0) return (int)cudaErrorNotSupported;
  const size_t smem = ptile_bytes(k.I);
  {
    cudaError_t e = ensure_smem((const void*)k_dtkp_apply<K, WT, AR>, smem);
    if (e != cudaSuccess) return (int)e;
  }
  // one resident wave of CTAs (x: 32-sample columns, y: strided over the work blocks)
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dtkp_apply<K, WT, AR>, 128, smem);
  const int64_t gx = ceil_div(k.B, kWarp);
  const int64_t resident = (int64_t)std::max(occ, 1) * std::max(sms, 1) * (k.sched ? 1 : SG_DTKP_WAVES);
  int gy;
  if (k.sched != nullptr) {
    // dynamic item schedule: one resident wave, no more warps than items
    gy = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(resident, gx), ceil_div((int64_t)k.n_items, 4)));
  } else {
    gy = (int)std::max<int64_t>(1, std::min<int64_t>(n_blocks, ceil_div(resident, gx)));
  }
  DtkpK kk = k;
  kk.n_blk = n_blocks;
  dim3 grid((unsigned)gx, gy);
  count_launch();
  k_dtkp_apply<K, WT, AR><<<grid, 128, smem, st>>>(kk);
  SG_LAUNCH_CHECK();
  return 0;
}

template <int K, int WT>
static int launch_apply_kw(const DtkpK& k, int n_blocks, cudaStream_t st) {
  if (k.arity == 1 && k.fused) return launch_apply_kwa<K, WT, 3>(k, n_blocks, st);
  if (k.arity == 1) return launch_apply_kwa<K, WT, 1>(k, n_blocks, st);
  if (k.arity == 2) return launch_apply_kwa<K, WT, 2>(k, n_blocks, st);
  return launch_apply_kwa<K, WT, 0>(k, n_blocks, st);
}

template <int K>
static int launch_apply_k(const DtkpK& k, int n_blocks, cudaStream_t st) {
  if (k.W <= 1) return launch_apply_kw<K, 1>(k, n_blocks, st);
  if (k.W <= 2) return launch_apply_kw<K, 2>(k, n_blocks, st);
  if (k.W <= 4) return launch_apply_kw<K, 4>(k, n_blocks, st);
  if (k.W <= 8) return launch_apply_kw<K, 8>(k, n_blocks, st);
  return (int)cudaErrorNotSupported;
}

// One launcher per K, defined in dtkp_apply_k.cu (compiled once per K value).
int launch_apply_K1(const DtkpK&, int, cudaStream_t);
int launch_apply_K2(const DtkpK&, int, cudaStream_t);
int launch_apply_K3(const DtkpK&, int, cudaStream_t);
int launch_apply_K4(const DtkpK&, int, cudaStream_t);
int launch_apply_K5(const DtkpK&, int, cudaStream_t);
int launch_apply_K6(const DtkpK&, int, cudaStream_t);
int launch_apply_K7(const DtkpK&, int, cudaStream_t);
int launch_apply_K8(const DtkpK&, int, cudaStream_t);

}  // namespace sg
