// K3 input ordering for the thread-sequential bulk pass.
//
// A warp of the bulk pass runs 32 inputs, one per lane; lanes whose inputs take
// different paths through the simulated kernel serialize (measured: 6.5 of 32
// lanes active on C2).  Inputs whose scalar arguments and array shapes agree
// take the same path unless array contents steer it, and most children share
// them with their parent (1-3 of n args mutated).  sfg_order buckets the round's
// inputs by a hash of that signature (counting sort with warp-aggregated
// atomics) and the bulk pass fetches inputs in bucket order.  Only the
// schedule changes: every input still writes its own verdict and edge row.
//
// The signature covers only the arguments that can steer control flow: a
// flow-insensitive taint analysis of the simulated kernels (control_arg_mask,
// abi.cu) marks the parameters reaching a setp, directly or through
// arithmetic, conversions or load addresses.  Arguments used only as strides
// or data (matmul's lda/ldb/ldc, array contents) move the stop point at most.
// i32 arguments enter by magnitude class (sign, bit length) rather than value:
// loop bounds of similar size run similar trip counts, and the inputs that will
// run long (huge bounds) end up in the same warps instead of one per warp.
#include "common.cuh"

namespace {

constexpr int kOrderBuckets = 4096;

SFG_DEV uint64_t sig_mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  return h * 0xBF58476D1CE4E5B9ull;
}

SFG_DEV int sig_bucket(const sfg_prog& P, const sfg_val* v, uint32_t mask) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (int a = 0; a < P.n_args; ++a) {
    if (!((mask >> a) & 1u)) continue;
    h = sig_mix(h, (uint64_t)v[a].kind | ((uint64_t)v[a].space << 8) | ((uint64_t)v[a].elem << 16));
    if (v[a].kind == SFG_V_I32) {
      // magnitude class (sign, bit length): loop bounds of similar size share a
      // bucket, so the long-running inputs gather in the same warps
      const int32_t x = (int32_t)v[a].bits;
      const uint32_t mag = x < 0 ? (uint32_t)(-(int64_t)x) : (uint32_t)x;
      h = sig_mix(h, ((uint64_t)(x < 0) << 8) | (uint64_t)(32 - __clz(mag)));
    } else if (v[a].kind != SFG_V_ARR) {
      h = sig_mix(h, v[a].bits);
    } else {
      h = sig_mix(h, v[a].nbytes);
      h = sig_mix(h, (uint64_t)v[a].size_override);
      h = sig_mix(h, (uint64_t)v[a].base_offset);
    }
  }
  return (int)((h >> 40) % kOrderBuckets);
}

// lanes of a warp that hit the same bucket add once (warp-aggregated atomics);
// returns this lane's slot in its bucket's run
SFG_DEV int warp_agg_add(int* counters, int bucket, bool active) {
  const unsigned act = __ballot_sync(0xffffffffu, active);
  if (!active) return 0;
  const unsigned peers = __match_any_sync(act, bucket);
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == leader) base = atomicAdd(&counters[bucket], __popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + __popc(peers & ((1u << lane) - 1u));
}

}  // namespace

extern "C" __global__ void sfg_order_hist_kernel(sfg_prog P, const sfg_val* vals, int n, uint32_t mask, int* hist,
                                                 int* sig, const int32_t* rep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n && (rep == nullptr || rep[i] == i);   // duplicates are not executed
  const int b = active ? sig_bucket(P, vals + (size_t)i * P.n_args, mask) : 0;
  if (active) sig[i] = b;
  warp_agg_add(hist, b, active);
}

// exclusive scan of the kOrderBuckets counts by one small CTA (128 threads x 32
// buckets): it must find room on SMs busy with other rounds' long inputs
extern "C" __global__ void __launch_bounds__(128) sfg_order_scan_kernel(int* hist, int* n_live) {
  __shared__ int part[128];
  constexpr int per = kOrderBuckets / 128;
  const int t = threadIdx.x;
  int s = 0;
  for (int k = 0; k < per; ++k) s += hist[t * per + k];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 128; off <<= 1) {
    const int v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = part[t] - s;
  for (int k = 0; k < per; ++k) {
    const int c = hist[t * per + k];
    hist[t * per + k] = run;
    run += c;
  }
  if (n_live && t == 127) *n_live = run;   // inputs in the schedule (executed)
}

extern "C" __global__ void sfg_order_scatter_kernel(int n, const int* sig, int* offs, int32_t* order,
                                                    const int32_t* rep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n && (rep == nullptr || rep[i] == i);
  const int b = active ? sig[i] : 0;
  const int pos = warp_agg_add(offs, b, active);
  if (active) order[pos] = i;
}

// ---------------------------------------------------------------------------
// Duplicate inputs of a round.  A COMPUTE phase is a pure function of the input's
// argument values and array bytes (the post-INIT image is shared; alloc ids are
// encoded relative to the input; the iteration only labels reports), and a child's
// values and bytes are a pure function of its parent and its ops (distinct
// arguments, so their order does not matter; rotation-count effects are recorded
// in the op).  Children with the same parent and the same set of ops therefore run
// identically: with a one-entry corpus ~half of a 2^18-input round repeats an
// earlier child.  sfg_dedupe_kernel maps every input to a representative (open
// addressing on a 32-bit hash of the child record's parent + ops, every match
// verified field by field -- a collision only costs a second execution, and equal
// children reached through different ops simply both run); only representatives
// are scheduled (sfg_order) and executed; sfg_dup_fill copies their verdicts and
// edge rows to the duplicates.
namespace {

SFG_DEV bool same_op(const sfg_op& x, const sfg_op& y) {
  return x.kind == y.kind && x.arg == y.arg && x.sub == y.sub && x.byte == y.byte && x.inner == y.inner &&
         x.isub == y.isub && x.ibyte == y.ibyte && x.mask == y.mask && x.imask == y.imask && x.index == y.index &&
         x.delta == y.delta;
}

SFG_DEV uint64_t op_hash(const sfg_op& x) {
  uint64_t h = sig_mix(0x510E527FADE682D1ull, (uint64_t)x.kind | ((uint64_t)x.arg << 8) | ((uint64_t)x.sub << 16) |
                                                  ((uint64_t)x.byte << 24) | ((uint64_t)x.inner << 32) |
                                                  ((uint64_t)x.isub << 40) | ((uint64_t)x.ibyte << 48));
  h = sig_mix(h, (uint64_t)x.mask | ((uint64_t)x.imask << 32));
  h = sig_mix(h, (uint64_t)x.index);
  return sig_mix(h, (uint64_t)x.delta);
}

// order-independent over the ops (a sum of per-op hashes), then mixed with the parent
SFG_DEV uint64_t dup_hash(const sfg_child& c) {
  uint64_t s = 0;
  for (int k = 0; k < c.n_ops; ++k) s += op_hash(c.ops[k]);
  return sig_mix(sig_mix(0x6A09E667F3BCC909ull, (uint64_t)(uint32_t)(c.parent < 0 ? 0 : c.parent) |
                                                    ((uint64_t)c.n_ops << 32)), s);
}

SFG_DEV bool same_input(const sfg_child& a, const sfg_child& b) {
  if ((a.parent < 0 ? 0 : a.parent) != (b.parent < 0 ? 0 : b.parent) || a.n_ops != b.n_ops) return false;
  for (int k = 0; k < a.n_ops; ++k) {   // every op of a is an op of b (ops touch distinct arguments)
    bool found = false;
    for (int j = 0; j < b.n_ops; ++j) found |= same_op(a.ops[k], b.ops[j]);
    if (!found) return false;
  }
  return true;
}

}  // namespace

// rep[i]: the input that runs for input i (itself, or an equal input whose verdict it
// takes).  table: `slots` 64-bit words, zeroed here; slot = hash32 << 32 | (index + 1).
extern "C" __global__ void sfg_dedupe_kernel(sfg_prog P, int n, const sfg_child* children, const sfg_val* vals,
                                             unsigned long long* table, int slots, int32_t* rep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sfg_child& c = children[i];
  const uint64_t h = dup_hash(c);
  const uint32_t h32 = (uint32_t)(h >> 32) | 1u;
  const unsigned long long mine = ((unsigned long long)h32 << 32) | (unsigned long long)(i + 1);
  int r = i;
  uint32_t s = (uint32_t)h & (uint32_t)(slots - 1);
  for (int probe = 0; probe < 64; ++probe) {
    // read first: a popular input's thousands of duplicates compare against the slot
    // without queueing atomics on it; only an empty slot is claimed
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(&table[s]);
    if (old == 0ull) {
      old = atomicCAS(&table[s], 0ull, mine);
      if (old == 0ull) break;   // first of its kind: runs itself
    }
    if ((uint32_t)(old >> 32) == h32) {
      const int j = (int)(old & 0xFFFFFFFFull) - 1;
      if (same_input(children[j], c)) {
        r = j;
        break;
      }
    }
    s = (s + 1) & (uint32_t)(slots - 1);
  }
  rep[i] = r;
}

// duplicates take their representative's verdict and edge row (after every pass ran)
extern "C" __global__ void sfg_dup_fill_kernel(int n, int n_edges, const int32_t* rep, sfg_verdict* verdicts,
                                               uint32_t* edge_counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = rep[i];
  if (r == i) return;
  verdicts[i] = verdicts[r];
  for (int e = 0; e < n_edges; ++e) edge_counts[(size_t)i * n_edges + e] = edge_counts[(size_t)r * n_edges + e];
}

// ---------------------------------------------------------------------------
// Grouped schedule: every input runs, each representative (sfg_dedupe) directly
// followed by its duplicates, representatives in sfg_order's signature order.  A
// warp of the bulk pass then takes runs of equal inputs: lanes that follow the same
// path through the simulated kernel on the same parent bytes issue together.
// cnt / fill: zeroed int32[n]; w: int64[n] (w[j] = 1 + duplicates of the j-th
// scheduled representative, 0 past n_live), scanned into start by the caller.
extern "C" __global__ void sfg_dup_count_kernel(int n, const int32_t* rep, int32_t* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool dup = i < n && rep[i] != i;
  warp_agg_add(cnt, dup ? rep[i] : 0, dup);
}

extern "C" __global__ void sfg_group_weights_kernel(int n, const int32_t* order, const int32_t* n_live,
                                                    const int32_t* cnt, int64_t* w) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  w[j] = j < *n_live ? 1 + (int64_t)cnt[order[j]] : 0;
}

extern "C" __global__ void sfg_group_place_kernel(int n, const int32_t* order, const int32_t* n_live,
                                                  const int64_t* start, int32_t* full, int32_t* rpos) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || j >= *n_live) return;
  const int r = order[j];
  full[start[j]] = r;
  rpos[r] = (int32_t)start[j];
}

extern "C" __global__ void sfg_group_dups_kernel(int n, const int32_t* rep, const int32_t* rpos, int32_t* fill,
                                                 int32_t* full) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool dup = i < n && rep[i] != i;
  const int r = dup ? rep[i] : 0;
  const int k = warp_agg_add(fill, r, dup);
  if (dup) full[rpos[r] + 1 + k] = i;
}

