// K1: batched type-aware mutation (schedule + op generation + payload apply).
//
// One fuzz input per thread for the draw-bound parts, one warp per input for
// the byte-moving part.  Every draw comes from the input's own numpy-compatible
// Philox stream (seed, keybase + it), so the child of input `it` is a pure
// function of (corpus at round start, rotation counts prefix, it):
//
//   sfg_plan_kernel    schedule_next (campaign.py:593-603) + the op-count and
//                      distinct-arg picks of mutate_testcase (mutation.py:502-511);
//                      emits per-int-arg pick flags for the rotation-count scan
//   sfg_mutate_kernel  re-derives the plan, then generate_op/apply_op per pick
//                      (mutation.py:371-496, 258-365) at descriptor level,
//                      child rng_seed = u64() (mutation.py:518), work layout
//   sfg_apply_kernel   parent payload -> child work region with the data-level
//                      ops applied (array_extreme/array_dim/array_elem), zero
//                      fill up to the materialized size (campaign.py:440-450)
//   sfg_regen_kernel   same payload rule, pristine bytes into a caller arena
//                      (admitted children -> corpus, first crashes -> host)
#include "common.cuh"
#include "philox.cuh"

namespace {

constexpr double kTypeAware = 0.4;  // mutation.py:51
// stream words kept per thread in shared memory (SfgWordStream): a child draws
// ~6-9 words on average, at most ~25 in practice (later words are recomputed)
constexpr uint32_t kMutateWords = 24;
constexpr uint32_t kPlanWords = 8;   // parent pick + op count + picks
__constant__ int32_t kIntDeltas[8] = {-16, -4, -2, -1, 1, 2, 4, 16};
// f32 bit patterns of _ARITH_DELTAS (1.0, -1.0, 0.5, 2.0, 1024.0, 0.001), mutation.py:55
__constant__ uint32_t kArith[6] = {0x3F800000u, 0xBF800000u, 0x3F000000u,
                                   0x40000000u, 0x44800000u, 0x3A83126Fu};

// Stream::weighted_choice over schedule_next's weights (rng.py:61-71).
template <class Strm>
__device__ int pick_parent(Strm& s, const sfg_prog& P, const CorpusView& C, int64_t it) {
  if (P.fanout > 0) return (int)(((it - 1) / P.fanout) % C.n);  // fixed fan-out: no draw
  const double x0 = s.random();
  // recent entries are a suffix of the non-seed entries (appended in admission order)
  int lo = C.n_seeds, hi = C.n;
  const int64_t cut = it - (int64_t)P.window;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (C.meta[mid].admitted_iteration >= cut) hi = mid; else lo = mid + 1;
  }
  const int64_t A = lo;             // weight-1 entries
  const int64_t Rn = C.n - lo;      // recent entries, weight w
  const double w = P.recent_weight;
  const bool exact = (w == floor(w)) && w >= 0.0 && (double)A + w * (double)Rn < 9007199254740992.0;
  if (exact) {
    const double total = (double)A + w * (double)Rn;
    const double x = x0 * total;
    if (x < (double)A) return (int)floor(x);
    if (Rn == 0 || w == 0.0) return C.n - 1;
    int64_t j = (int64_t)floor((x - (double)A) / w);
    if (j < 0) j = 0;
    while (j > 0 && !(x >= (double)A + w * (double)j)) --j;
    while (j < Rn && x >= (double)A + w * (double)(j + 1)) ++j;
    return j >= Rn ? C.n - 1 : (int)(A + j);
  }
  double total = 0.0;
  for (int i = 0; i < C.n; ++i) total += (i < A) ? 1.0 : w;
  const double x = x0 * total;
  double acc = 0.0;
  for (int i = 0; i < C.n; ++i) {
    acc += (i < A) ? 1.0 : w;
    if (x < acc) return i;
  }
  return C.n - 1;
}

// mutate_testcase picks (mutation.py:502-511)
template <class Strm>
__device__ int draw_picks(Strm& s, const sfg_prog& P, int8_t* picks) {
  int cap = P.max_ops < P.n_mutable ? P.max_ops : P.n_mutable;
  const int n_ops = 1 + s.geometric_small(0.5, cap - 1);
  // pool.pop(integers(len)): the idx-th remaining entry of mutable_args, kept as a
  // bitmask of remaining positions (registers, no local array)
  int len = P.n_mutable;
  uint32_t rem = len >= 32 ? 0xffffffffu : (1u << len) - 1u;
  for (int k = 0; k < n_ops; ++k) {
    const int idx = (int)s.integers(0, len);
    const int pos = (int)__fns(rem, 0, idx + 1);
    picks[k] = P.mutable_args[pos];
    rem &= ~(1u << pos);
    --len;
  }
  return n_ops;
}

template <class Strm>
__device__ void gen_int_byte(Strm& s, sfg_op& op) {  // mutation.py:396-401
  op.kind = SFG_M_INT_BYTE;
  if (s.random() < 0.5) {
    op.sub = 0;
    op.byte = (uint8_t)s.integers(0, 4);
    op.mask = (uint32_t)s.integers(1, 256);
  } else {
    op.sub = 1;
    op.delta = kIntDeltas[s.integers(0, 8)];
  }
}

template <class Strm>
__device__ void gen_float_op(Strm& s, sfg_op& op) {  // mutation.py:404-422
  if (s.random() < kTypeAware) {
    const int pick = (int)s.integers(0, 4);
    if (pick == 0) {
      op.kind = SFG_M_FLOAT_SIGN;
    } else if (pick == 1) {
      op.kind = SFG_M_FLOAT_EXPONENT;
      op.sub = (uint8_t)s.integers(0, 3);  // ones, zeros, bit
      if (op.sub == 2) op.byte = (uint8_t)s.integers(0, 8);
    } else if (pick == 2) {
      op.kind = SFG_M_FLOAT_MANTISSA;
      op.mask = (uint32_t)s.integers(1, 1 << 23);
    } else {
      op.kind = SFG_M_FLOAT_ARITH;
      op.mask = kArith[s.integers(0, 6)];
    }
    return;
  }
  op.kind = SFG_M_FLOAT_BYTE;
  op.byte = (uint8_t)s.integers(0, 4);
  op.mask = (uint32_t)s.integers(1, 256);
}

// _offset_palette (mutation.py:425-438): sorted distinct magnitudes in (0, 2*size], +m then -m
template <class Strm>
__device__ int64_t offset_choice(Strm& s, const sfg_prog& P, uint64_t nbytes) {
  const int64_t g = P.mut_granule, rz = P.mut_redzone;
  const int64_t size = (int64_t)nbytes > g ? (int64_t)nbytes : g;
  int64_t m[11] = {g, 2 * g, rz, rz + g, 2 * rz, 2 * rz + g, 2 * rz - g, size, size + 2 * rz,
                   size + rz, 2 * size};
  // sort + dedupe + keep (0, 2*size]: a rare path, kept small (not unrolled)
#pragma unroll 1
  for (int i = 1; i < 11; ++i) {  // insertion sort
    const int64_t v = m[i];
    int j = i - 1;
#pragma unroll 1
    while (j >= 0 && m[j] > v) { m[j + 1] = m[j]; --j; }
    m[j + 1] = v;
  }
  int64_t u[11];
  int n = 0;
#pragma unroll 1
  for (int i = 0; i < 11; ++i)
    if (m[i] > 0 && m[i] <= 2 * size && (n == 0 || u[n - 1] != m[i])) u[n++] = m[i];
  if (n == 0) {
    const int64_t k = s.integers(0, 2);
    return k ? -g : g;
  }
  const int64_t k = s.integers(0, 2 * n);
  return (k & 1) ? -u[k >> 1] : u[k >> 1];
}

template <class Strm>
__device__ void space_choice(Strm& s, uint8_t cur, sfg_op& op) {
  uint8_t others[2];
  int n = 0;
  for (uint8_t sp = 0; sp < 3; ++sp)
    if (sp != cur) others[n++] = sp;
  op.sub = others[s.integers(0, 2)];
}

template <class Strm>
__device__ void gen_array_op(Strm& s, const sfg_prog& P, const sfg_val& v, sfg_op& op) {
  if (v.count == 0) {  // mutation.py:443-450
    const int pick = (int)s.integers(0, 3);
    if (pick == 0) {
      op.kind = SFG_M_ARRAY_DIM; op.sub = 1; op.mask = 4;
    } else if (pick == 1) {
      op.kind = SFG_M_PTR_SPACE; space_choice(s, v.space, op);
    } else {
      op.kind = SFG_M_PTR_OFFSET; op.delta = offset_choice(s, P, v.nbytes);
    }
    return;
  }
  if (s.random() < kTypeAware) {  // mutation.py:451-464
    const int pick = (int)s.integers(0, 5);
    if (pick == 0) {
      op.kind = SFG_M_ARRAY_EXTREME; op.sub = (uint8_t)s.integers(0, 3);
    } else if (pick == 1) {  // _gen_extents (mutation.py:477-487)
      op.kind = SFG_M_ARRAY_DIM;
      const uint32_t n = v.count;
      if (n >= 2) {
        const int nopt = (n % 2 == 0) ? 3 : 2;
        const int k = (int)s.integers(0, nopt);
        if (k == 0) { op.sub = 1; op.mask = n / 2; }
        else if (k == 1) { op.sub = 2; op.mask = n; op.imask = 2; }
        else { op.sub = 2; op.mask = 2; op.imask = n / 2; }
      } else {
        s.integers(0, 1);  // choice of a one-element list draws nothing (rng == 0)
        op.sub = 1; op.mask = 2 * n + 2;
      }
    } else if (pick == 2) {
      op.kind = SFG_M_ARRAY_EMPTY;
    } else if (pick == 3) {
      op.kind = SFG_M_PTR_SPACE; space_choice(s, v.space, op);
    } else {
      op.kind = SFG_M_PTR_OFFSET; op.delta = offset_choice(s, P, v.nbytes);
    }
    return;
  }
  op.kind = SFG_M_ARRAY_ELEM;  // mutation.py:465-474
  op.index = (uint32_t)s.integers(0, (int64_t)v.count);
  sfg_op in{};
  if (v.elem == 1) {
    do { in = sfg_op{}; gen_float_op(s, in); } while (in.kind == SFG_M_FLOAT_ARITH);
  } else {
    gen_int_byte(s, in);
  }
  op.inner = in.kind; op.isub = in.sub; op.ibyte = in.byte; op.imask = in.mask; op.delta = in.delta;
}

// descriptor-level apply_op (mutation.py:258-357); payload bytes are done by emit_child
__device__ void apply_desc(const sfg_prog& P, sfg_val& v, const sfg_op& op) {
  switch (op.kind) {
    case SFG_M_INT_BOUNDARY:
    case SFG_M_INT_BYTE: v.bits = int_bits_op(v.bits, op.kind, op.sub, op.byte, op.mask, op.delta); break;
    case SFG_M_FLOAT_SIGN: case SFG_M_FLOAT_EXPONENT: case SFG_M_FLOAT_MANTISSA:
    case SFG_M_FLOAT_BYTE: case SFG_M_FLOAT_ARITH:
      v.bits = float_bits_op(v.bits, op.kind, op.sub, op.byte, op.mask); break;
    case SFG_M_ARRAY_EXTREME: v.nbytes = 4u * v.count; break;
    case SFG_M_ARRAY_DIM:
      v.ndim = op.sub; v.ext[0] = op.mask; v.ext[1] = op.sub == 2 ? op.imask : 0; v.ext[2] = v.ext[3] = 0;
      v.count = op.sub == 2 ? op.mask * op.imask : op.mask;
      v.nbytes = 4u * v.count;
      break;
    case SFG_M_ARRAY_EMPTY: v.ndim = 1; v.ext[0] = v.ext[1] = v.ext[2] = v.ext[3] = 0; v.count = 0; v.nbytes = 0; break;
    case SFG_M_PTR_SPACE: v.space = op.sub; break;
    case SFG_M_PTR_OFFSET: {
      const int64_t lim = 2 * (int64_t)(v.nbytes > 4 ? v.nbytes : 4);
      const int64_t d = op.delta < -lim ? -lim : (op.delta > lim ? lim : op.delta);
      v.base_offset += d;
      break;
    }
    default: break;  // ARRAY_ELEM: payload only
  }
}

}  // namespace

extern "C" __global__ void sfg_plan_kernel(sfg_prog P, CorpusView C, int64_t it0, int n,
                                           int32_t* parent_out, int8_t* picks_out, uint32_t* flags_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t it = it0 + i;
  int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
  int parent = -1;
  __shared__ uint64_t words[kPlanWords * 128];
  if (it != 1) {
    SfgWordStream s;
    s.init(words + threadIdx.x, 128, kPlanWords, P.master_seed, P.keybase + (uint64_t)it);
    parent = pick_parent(s, P, C, it);
    draw_picks(s, P, picks);
  }
  parent_out[i] = parent;
  for (int k = 0; k < SFG_MAX_OPS; ++k) picks_out[i * SFG_MAX_OPS + k] = picks[k];
  for (int c = 0; c < P.n_int_args; ++c) flags_out[(size_t)i * P.n_int_args + c] = 0;
  for (int k = 0; k < SFG_MAX_OPS; ++k)
    if (picks[k] >= 0 && P.int_slot[picks[k]] >= 0) flags_out[(size_t)i * P.n_int_args + P.int_slot[picks[k]]] = 1;
}

// counts_prefix[i][c]: rotation count of int column c seen by input i
// One child of the mutation stage (mutation.py:499-518 mutate_testcase + the
// work layout): parent pick, picks, op generation, descriptor-level apply, child
// values written once.  s: the input's Philox stream (its own in the batched
// contract, the worker's in the sequential one); cnt_of[c] + (cnt_pre ? cnt_pre[c] : 0):
// MutationSchedule rotation count of int column c as this input sees it (read
// where a pick needs it: no per-thread array); picks out.
// EMIT = false: the draws only (the sequential discipline's candidate walker,
// seqgen): nothing is written, the stream ends where the child's draws end.
// cnt_of == nullptr: rotation counts saturated (every mutable int column >= 3).
template <bool EMIT = true, class Strm>
__device__ __forceinline__ void mutate_child(const sfg_prog& P, const CorpusView& C, int64_t it, Strm& s,
                                             const uint64_t* cnt_of, const uint64_t* cnt_pre, int8_t* picks,
                                             sfg_child& ch,
                                             sfg_val* __restrict__ vout) {
  if (EMIT) {
    memset(&ch, 0, sizeof(ch));
    ch.it = it;
  }
  const sfg_val* __restrict__ pv = C.vals;   // parent values (the seed for it == 1)
  // picked args: the mutated value goes straight to vout; its kind / materialized
  // size / nbytes stay in registers for the layout pass
  int ma[SFG_MAX_OPS] = {-1, -1, -1};
  uint64_t msz[SFG_MAX_OPS] = {0, 0, 0};
  uint32_t mnb[SFG_MAX_OPS] = {0, 0, 0};
  uint8_t mkind[SFG_MAX_OPS] = {0, 0, 0};
  if (it == 1) {  // fuzz_loop evaluates the recorded seed first (campaign.py:739-740)
    if (!EMIT) return;
    ch.parent = -1;
    ch.rng_seed = C.meta[0].rng_seed;
  } else {
    const int parent = pick_parent(s, P, C, it);
    const int n_ops = draw_picks(s, P, picks);
    if (EMIT) {
      ch.parent = parent;
      ch.n_ops = n_ops;
    }
    pv = C.vals + (size_t)parent * P.n_args;
    for (int k = 0; k < n_ops; ++k) {
      const int a = picks[k];
      sfg_op op;
      memset(&op, 0, sizeof(op));
      op.arg = (uint8_t)a;
      sfg_val v = pv[a];
      if (v.kind == SFG_V_I32) {  // MutationSchedule.next_int_op (mutation.py:378-386)
        const int c = P.int_slot[a];
        const uint64_t cnt = cnt_of ? cnt_of[c] + (cnt_pre ? cnt_pre[c] : 0ull) : 3ull;
        if (cnt < 3) {
          op.kind = SFG_M_INT_BOUNDARY;
          op.sub = (uint8_t)cnt;
        } else if (s.random() < kTypeAware) {
          op.kind = SFG_M_INT_BOUNDARY;
          op.sub = (uint8_t)s.integers(0, 3);
        } else {
          gen_int_byte(s, op);
        }
      } else if (v.kind == SFG_V_F32) {
        gen_float_op(s, op);
      } else {
        gen_array_op(s, P, v, op);
      }
      if (EMIT) {
        apply_desc(P, v, op);
        vout[a] = v;   // data_off filled by the layout pass
        ma[k] = a;
        msz[k] = sfg_mat_size(v);
        mnb[k] = v.nbytes;
        mkind[k] = v.kind;
        ch.ops[k] = op;
      }
    }
    const uint64_t seed = s.next64();
    if (!EMIT) return;
    ch.rng_seed = seed;
  }
  // one pass over the child's values: parent value or its mutation, work layout
  // (array regions at materialized size, 16-aligned, then COMPUTE named allocs),
  // readout sizes; each value written once
  uint64_t off = 0, pri = 0, rb = P.diff_readback ? (uint64_t)P.readout_bytes_fixed : 0ull;
  for (int a = 0; a < P.n_args; ++a) {
    int m = -1;
#pragma unroll
    for (int k = 0; k < SFG_MAX_OPS; ++k)
      if (ma[k] == a) m = k;
    uint32_t nb;
    if (m >= 0) {       // mutated: value already written
      nb = mnb[m];
      if (mkind[m] == SFG_V_ARR) {
        vout[a].data_off = off;
        off += sfg_align16(msz[m]);
      }
    } else {
      sfg_val v = pv[a];
      nb = v.nbytes;
      if (v.kind == SFG_V_ARR) {
        v.data_off = off;
        off += sfg_align16(sfg_mat_size(v));
      }
      vout[a] = v;
    }
    if (P.diff_readback)
      for (int k = 0; k < P.n_copyout_arg; ++k)
        if (P.copyout_arg[k] == a) rb += sfg_align16(nb);
    if ((P.copy_src_mask >> a) & 1u) pri += sfg_align16(nb);
  }
  ch.work_bytes = off + (uint64_t)P.named_work_bytes + sfg_ov_bytes(P.ov_cap) + pri;
  ch.readout_bytes = rb;
  ch.readout_bytes = rb;
}

extern "C" __global__ void __launch_bounds__(128, 8) sfg_mutate_kernel(sfg_prog P, CorpusView C, int64_t it0, int n,
                                             const uint64_t* counts_prefix, const uint64_t* counts_base,
                                             sfg_child* child_out, sfg_val* vals_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t it = it0 + i;
  __shared__ uint64_t words[kMutateWords * 128];
  SfgWordStream s;
  s.init(words + threadIdx.x, 128, kMutateWords, P.master_seed, P.keybase + (uint64_t)it);
  int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
  sfg_child ch;   // assembled locally, stored once (child_out stores would alias the parent reads)
  mutate_child(P, C, it, s, counts_base, counts_prefix ? counts_prefix + (size_t)i * P.n_int_args : nullptr, picks,
               ch, vals_out + (size_t)i * P.n_args);
  child_out[i] = ch;
}

// The reference fuzz_loop's own stream discipline (campaign.py:714-749): one worker
// stream Stream(master_seed, 1000 + w) and one MutationSchedule consumed input after
// input.  A single thread generates the round's children in order from the worker
// state (*state), saving the state before every input (states[0..n]) and the
// int-arg picks (flags, as sfg_plan) so the host can cut the round after an
// admission and resume exactly there.  Rotation counts start from counts_base.
extern "C" __global__ void sfg_plan_seq_kernel(sfg_prog P, CorpusView C, int64_t it0, int n, const SfgStream* state,
                                               const uint64_t* counts_base, sfg_child* child_out, sfg_val* vals_out,
                                               uint32_t* flags_out, SfgStream* states) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  SfgStream s = *state;
  uint64_t cnt[SFG_MAX_ARGS];
  for (int c = 0; c < P.n_int_args && c < SFG_MAX_ARGS; ++c) cnt[c] = counts_base[c];
  for (int i = 0; i < n; ++i) {
    states[i] = s;
    const int64_t it = it0 + i;
    int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
    sfg_child ch;
    mutate_child(P, C, it, s, cnt, nullptr, picks, ch, vals_out + (size_t)i * P.n_args);
    child_out[i] = ch;
    for (int c = 0; c < P.n_int_args; ++c) flags_out[(size_t)i * P.n_int_args + c] = 0;
    for (int k = 0; k < SFG_MAX_OPS; ++k)
      if (picks[k] >= 0 && P.int_slot[picks[k]] >= 0) {
        flags_out[(size_t)i * P.n_int_args + P.int_slot[picks[k]]] = 1;
        ++cnt[P.int_slot[picks[k]]];
      }
  }
  states[n] = s;
}

// ---------------------------------------------------------------------------
// Sequential discipline in parallel (seqgen).  The reference fuzz_loop draws every
// child from ONE worker stream (campaign.py:714-749): child k starts where child
// k-1's draws ended, and how many words a child draws is data dependent.  The
// round's children are found without walking the stream one child at a time:
//
//   * a stream position at a child boundary is (w, has32, cache32): w words
//     consumed, and the cached high half of the last odd next32 draw.  Every op
//     generator ends on a next32 and every child on rng_seed = next64, so at a
//     boundary the cache is empty or holds the high half of word w-2.  The
//     candidates are x = 2 (w - w0) + h, h = 1 for "cache = hi32(word w-2)", over
//     the round's word range [w0, w0 + W).
//   * sfg_seq_walk: every candidate draws one child (draws only) and records its
//     successor candidate (kSeqEscape: the end state is not a candidate,
//     kSeqOut: beyond the range);
//   * sfg_seq_jump: pointer doubling, J_{k+1} = J_k o J_k;
//   * sfg_seq_path: top-down from the start, path[q0 + j + 2^k] = J_k[path[q0 + j]];
//   * sfg_seq_mutate: every child generated from its start position in parallel,
//     exactly as sfg_mutate does, with the stream state before every child
//     (states[], the resume points of a cut) and the int-arg picks.
//
// Exact when the round's children do not depend on their iteration number or on
// each other beyond the stream: rotation counts saturated (>= 3, mutation.py:378-
// 386), no fan-out, no corpus entry leaving the recent window inside the round
// (the host cuts rounds there), it0 >= 2.  The first child whose start is not a
// candidate (or out of range) truncates the round (stats[0] = valid children);
// the host cuts the round there and resumes from states[stats[0]], which the
// previous child's thread wrote from its exact end state.
constexpr int32_t kSeqEscape = -1;
constexpr int32_t kSeqOut = -2;
constexpr int kSeqWinBlocks = 24;   // Philox blocks per warp window (96 words)

__device__ __forceinline__ int32_t seq_candidate(uint64_t w, uint32_t has32, uint32_t cache32, uint64_t w0, int64_t W,
                                                 uint64_t hi_w2) {
  if (w - w0 >= (uint64_t)W) return kSeqOut;
  if (!has32) return (int32_t)(2 * (w - w0));
  return (w >= 2 && cache32 == (uint32_t)(hi_w2 >> 32)) ? (int32_t)(2 * (w - w0) + 1) : kSeqEscape;
}

extern "C" __global__ void __launch_bounds__(128) sfg_seq_walk_kernel(sfg_prog P, CorpusView C, int64_t it,
                                                                     const SfgStream* start, int64_t W,
                                                                     int32_t* next) {
  __shared__ uint64_t win[4][kSeqWinBlocks * 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t w0 = sfg_state_words(*start);
  const uint64_t key0 = start->key0, key1 = start->key1;
  const int64_t xw = (int64_t)blockIdx.x * 128 + warp * 32;   // the warp's first candidate
  const uint64_t wlo = w0 + (uint64_t)(xw / 2);
  const uint64_t wfirst = wlo >= 2 ? ((wlo - 2) & ~3ull) : 0ull;
  if (lane < kSeqWinBlocks) {
    const SfgPhilox4 o = sfg_philox4x64_10(wfirst / 4 + lane + 1, 0, 0, 0, key0, key1);
    win[warp][lane * 4] = o.v0;
    win[warp][lane * 4 + 1] = o.v1;
    win[warp][lane * 4 + 2] = o.v2;
    win[warp][lane * 4 + 3] = o.v3;
  }
  __syncwarp();
  const int64_t x = xw + lane;
  if (x >= 2 * W) return;
  SfgWinStream s;
  s.key0 = key0;
  s.key1 = key1;
  s.wlo = wfirst;
  s.swin = (uint32_t)__cvta_generic_to_shared(&win[warp][0]);
  s.nwin = kSeqWinBlocks * 4;
  s.w = w0 + (uint64_t)(x / 2);
  s.has32 = (uint32_t)(x & 1);
  if (s.has32 && s.w < 2) {
    next[x] = kSeqEscape;
    return;
  }
  s.cache32 = s.has32 ? (uint32_t)(s.word(s.w - 2) >> 32) : 0u;
  int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
  sfg_child unused;
  mutate_child<false>(P, C, it, s, nullptr, nullptr, picks, unused, nullptr);
  const uint64_t w2 = s.w;
  next[x] = seq_candidate(w2, s.has32, s.cache32, w0, W, (s.has32 && w2 >= 2) ? s.word(w2 - 2) : 0ull);
}

extern "C" __global__ void sfg_seq_jump_kernel(const int32_t* J, int32_t* J2, int64_t M) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < M; x += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = J[x];
    J2[x] = j < 0 ? j : J[j];
  }
}

// The round's first child: its start position is a candidate (q0 = 0, path[0]) or,
// when not, it is generated here from the exact state and the path starts at its
// successor (q0 = 1).  stats: [0] valid children, [1] words drawn by them.
extern "C" __global__ void sfg_seq_root_kernel(sfg_prog P, CorpusView C, int64_t it0, int n, const SfgStream* start,
                                               int64_t W, const uint64_t* counts_base, sfg_child* child_out,
                                               sfg_val* vals_out, uint32_t* flags_out, SfgStream* states,
                                               int32_t* path, int32_t* q0, unsigned long long* stats) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  SfgStream s = *start;
  const uint64_t w0 = sfg_state_words(s);
  states[0] = s;
  stats[0] = (unsigned long long)n;
  stats[1] = 0ull;
  const int32_t x0 = seq_candidate(w0, s.has32, s.cache32, w0, W,
                                   (s.has32 && w0 >= 2) ? sfg_stream_word(s.key0, s.key1, w0 - 2) : 0ull);
  if (x0 >= 0) {
    path[0] = x0;
    *q0 = 0;
    return;
  }
  int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
  sfg_child ch;
  mutate_child(P, C, it0, s, counts_base, nullptr, picks, ch, vals_out);
  child_out[0] = ch;
  for (int c = 0; c < P.n_int_args; ++c) flags_out[c] = 0;
  for (int k = 0; k < SFG_MAX_OPS; ++k)
    if (picks[k] >= 0 && P.int_slot[picks[k]] >= 0) flags_out[P.int_slot[picks[k]]] = 1;
  states[1] = s;
  const uint64_t w1 = sfg_state_words(s);
  stats[1] = w1 - w0;
  path[1] = seq_candidate(w1, s.has32, s.cache32, w0, W,
                          (s.has32 && w1 >= 2) ? sfg_stream_word(s.key0, s.key1, w1 - 2) : 0ull);
  if (path[1] < 0) stats[0] = 1ull;
  *q0 = 1;
}

// one level of the top-down path: path[q0 + j + step] = J[path[q0 + j]], j a multiple of 2 step
extern "C" __global__ void sfg_seq_path_kernel(const int32_t* J, int32_t* path, const int32_t* q0p, int n,
                                               int64_t step) {
  const int q0 = *q0p;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2 * step;
  if (j + step > (int64_t)n - q0) return;
  const int32_t v = path[q0 + j];
  path[q0 + j + step] = v < 0 ? v : J[v];
}

extern "C" __global__ void __launch_bounds__(128, 8) sfg_seq_mutate_kernel(
    sfg_prog P, CorpusView C, int64_t it0, int n, const SfgStream* start, const int32_t* path, const int32_t* q0p,
    const uint64_t* counts_base, sfg_child* child_out, sfg_val* vals_out, uint32_t* flags_out, SfgStream* states,
    unsigned long long* stats) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int q0 = *q0p;
  if (j < q0 || j >= n) return;
  const uint64_t w0 = sfg_state_words(*start);
  const uint64_t key0 = start->key0, key1 = start->key1;
  int32_t x = path[j];
  const bool valid = x >= 0;
  if (!valid) {   // past the truncation: any well-formed child (discarded by the cut)
    atomicMin(&stats[0], (unsigned long long)j);
    x = 0;
  }
  const uint64_t w = w0 + (uint64_t)(x / 2);
  const uint32_t h = (uint32_t)(x & 1);
  const uint32_t c = h ? (uint32_t)(sfg_stream_word(key0, key1, w - 2) >> 32) : 0u;
  if (valid) {
    SfgStream st;
    sfg_state_at(st, key0, key1, w, h, c);
    states[j] = st;
  }
  __shared__ uint64_t words[kMutateWords * 128];
  SfgWordStream s;
  s.init_at(words + threadIdx.x, 128, kMutateWords, key0, key1, w, h, c);
  int8_t picks[SFG_MAX_OPS] = {-1, -1, -1};
  sfg_child ch;
  mutate_child(P, C, it0 + j, s, counts_base, nullptr, picks, ch, vals_out + (size_t)j * P.n_args);
  child_out[j] = ch;
  for (int cc = 0; cc < P.n_int_args; ++cc) flags_out[(size_t)j * P.n_int_args + cc] = 0;
  if (valid)
    for (int k = 0; k < SFG_MAX_OPS; ++k)
      if (picks[k] >= 0 && P.int_slot[picks[k]] >= 0) flags_out[(size_t)j * P.n_int_args + P.int_slot[picks[k]]] = 1;
  if (valid) {
    const uint64_t w2 = s.words();
    atomicMax(&stats[1], (unsigned long long)(w2 - w0));
    if (j == n - 1 || path[j + 1] < 0) {   // the next start is not a candidate: its exact state
      SfgStream e;
      sfg_state_at(e, key0, key1, w2, s.has32, s.cache32);
      states[j + 1] = e;
    }
  }
}

// warp per input: parent payloads -> child work region (materialized contents)
// (sel != nullptr: only the inputs sel[0 .. *sel_n) -- the deferred long inputs
// re-materialized for the tail pass)
// An input's arrays are a few hundred bytes (16-byte chunks), so a group of
// kApplyLanes lanes handles one input and a warp keeps 32 / kApplyLanes inputs'
// dependent descriptor loads in flight at once.
constexpr int kApplyLanes = 8;

extern "C" __global__ void sfg_apply_kernel(sfg_prog P, CorpusView C, int n, const sfg_child* children,
                                            const sfg_val* vals, const uint64_t* work_base, uint8_t* work,
                                            const int32_t* sel, const int* sel_n) {
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / kApplyLanes;
  const int lane = threadIdx.x % kApplyLanes;
  const int ngroups = (gridDim.x * blockDim.x) / kApplyLanes;
  if (sel) n = *sel_n;
  for (int j = gid; j < n; j += ngroups) {
    const int i = sel ? sel[j] : j;
    const sfg_child& ch = children[i];
    const int parent = ch.parent < 0 ? 0 : ch.parent;
    const sfg_val* pv = C.vals + (size_t)parent * P.n_args;
    const sfg_val* cv = vals + (size_t)i * P.n_args;
    uint8_t* base = work + work_base[i];
    for (int a = 0; a < P.n_args; ++a) {
      if (cv[a].kind != SFG_V_ARR) continue;
      const sfg_op* op = nullptr;
      for (int k = 0; k < ch.n_ops; ++k)
        if (ch.ops[k].arg == a) op = &ch.ops[k];
      emit_child(base + cv[a].data_off, sfg_mat_size(cv[a]), C.data + pv[a].data_off, pv[a].nbytes, cv[a],
                 op, lane, kApplyLanes);
      if ((P.copy_src_mask >> a) & 1u)   // the test case's own bytes for copy_in (campaign.py:404-409)
        emit_child(base + sfg_pristine_off(&P, cv, ch.work_bytes, a, nullptr), cv[a].nbytes, C.data + pv[a].data_off,
                   pv[a].nbytes, cv[a], op, lane, kApplyLanes);
    }
  }
}

// warp per selected input: pristine child payloads into dst (dst_off per (selected, arg))
extern "C" __global__ void sfg_regen_kernel(sfg_prog P, CorpusView C, int n_sel, const int32_t* sel,
                                            const sfg_child* children, const sfg_val* vals,
                                            const uint64_t* dst_off, uint8_t* dst) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j = warp; j < n_sel; j += nwarps) {
    const int i = sel[j];
    const sfg_child& ch = children[i];
    const int parent = ch.parent < 0 ? 0 : ch.parent;
    const sfg_val* pv = C.vals + (size_t)parent * P.n_args;
    const sfg_val* cv = vals + (size_t)i * P.n_args;
    for (int a = 0; a < P.n_args; ++a) {
      if (cv[a].kind != SFG_V_ARR) continue;
      const sfg_op* op = nullptr;
      for (int k = 0; k < ch.n_ops; ++k)
        if (ch.ops[k].arg == a) op = &ch.ops[k];
      emit_child(dst + dst_off[(size_t)j * P.n_args + a], cv[a].nbytes, C.data + pv[a].data_off,
                 pv[a].nbytes, cv[a], op, lane, 32);
    }
  }
}
