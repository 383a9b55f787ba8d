// K4/K5: per-round triage, novelty, dedupe and corpus compaction, plus the
// device prefix scans the batched-round contract reduces to.
//
// The reference absorbs inputs one at a time (campaign.py:825-846): merge the
// input's edges into the global map, register its finding (FindingsLog.add,
// sanitizer.py:216-225), stop if the stop rule fires, else admit it when it
// hit an edge the global map had never seen.  Over a round of inputs in `it`
// order that is exactly:
//   stop   = min{i : finding(i) and stop-rule(i)}                (atomicMin)
//   first_hit[e] = min{i : i hit e}                              (warp min + atomicMin)
//   edge_total[e] += sum_{i<=stop} count_i(e)                    (warp sum + atomicAdd)
//   key_first[k] = min{i<=stop : key(i) = k}, key_count[k] += #  (match_any + atomics)
//   admit(i) = i<=stop, no finding, it!=1, exists e: count_i(e)>0,
//              e not in G_round_start, first_hit[e] == i
//   alloc ids of input i = round base + exclusive_scan(allocs)   (device scan)
#include "common.cuh"

namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
SFG_DEV uint64_t load_as_u64(const T* p, size_t idx) { return (uint64_t)p[idx]; }

SFG_DEV uint64_t block_exclusive_scan(uint64_t v, uint64_t* sh, uint64_t& total) {
  // warp scan then warp-sums scan (blockDim.x == kScanThreads)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    uint64_t s = lane < (kScanThreads / 32) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < (kScanThreads / 32)) sh[lane] = s;
  }
  __syncthreads();
  const uint64_t before = w ? sh[w - 1] : 0;
  total = sh[kScanThreads / 32 - 1];
  __syncthreads();
  return before + x - v;
}
}  // namespace

// ---- generic exclusive scan over a strided column: out[i] = sum_{j<i} in[j*stride + col]
template <typename T>
__global__ void sfg_scan_tiles(const T* in, int64_t n, int stride, int col, uint64_t* tile_sums) {
  __shared__ uint64_t sh[32];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint64_t s = 0;
  for (int k = 0; k < kScanItems; ++k)
    if (t0 + k < n) s += load_as_u64(in, (size_t)(t0 + k) * stride + col);
  uint64_t total;
  block_exclusive_scan(s, sh, total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void sfg_scan_tile_sums(uint64_t* tile_sums, int64_t ntiles, uint64_t* grand_total) {
  __shared__ uint64_t sh[32];
  uint64_t carry = 0;
  for (int64_t base = 0; base < ntiles; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const uint64_t v = i < ntiles ? tile_sums[i] : 0;
    uint64_t total;
    const uint64_t ex = block_exclusive_scan(v, sh, total);
    if (i < ntiles) tile_sums[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0 && grand_total) *grand_total = carry;
}

template <typename T>
__global__ void sfg_scan_apply(const T* in, int64_t n, int stride, int col, const uint64_t* tile_off,
                               uint64_t* out, int out_stride, int out_col) {
  __shared__ uint64_t sh[32];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = t0 + k < n ? load_as_u64(in, (size_t)(t0 + k) * stride + col) : 0;
    s += v[k];
  }
  uint64_t total;
  uint64_t run = tile_off[blockIdx.x] + block_exclusive_scan(s, sh, total);
  for (int k = 0; k < kScanItems; ++k) {
    if (t0 + k < n) out[(size_t)(t0 + k) * out_stride + out_col] = run;
    run += v[k];
  }
}

template __global__ void sfg_scan_tiles<uint32_t>(const uint32_t*, int64_t, int, int, uint64_t*);
template __global__ void sfg_scan_tiles<uint64_t>(const uint64_t*, int64_t, int, int, uint64_t*);
template __global__ void sfg_scan_apply<uint32_t>(const uint32_t*, int64_t, int, int, const uint64_t*, uint64_t*, int, int);
template __global__ void sfg_scan_apply<uint64_t>(const uint64_t*, int64_t, int, int, const uint64_t*, uint64_t*, int, int);

// ---- triage
// Indices are GLOBAL round indices g = i_base + i (a rank owns the contiguous
// slice [i_base, i_base + n) of the round), so the per-rank partials below
// merge across GPUs with plain MIN / SUM all-reduces; with
// one GPU i_base = 0 and the reductions are the identity.  "None" is
// INT32_MAX so that a signed MIN all-reduce is the merge.
constexpr int32_t kNone = 0x7fffffff;

// scalars[0] = stop index, scalars[1] = first fatal index
extern "C" __global__ void sfg_stop_kernel(sfg_prog P, const sfg_verdict* V, int n, int i_base, int32_t* scalars) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sfg_verdict& v = V[i];
  if (v.status >= SFG_ST_OUT_OF_SPACE) atomicMin(&scalars[1], i_base + i);
  if (v.status == SFG_ST_FINDING && (P.stop_first || v.bug_class == P.stop_class)) atomicMin(&scalars[0], i_base + i);
}

// per-round partials: first_hit[e] (MIN), edge_delta[e] (SUM), key_first/key_count
// (MIN/SUM), entered_cnt[kernel] (SUM; > 0 <=> entered), allocs per input
constexpr int kAbsorbEdges = 1024;   // SFG_MAX_EDGES: shared-memory combine of the CTA's warps

extern "C" __global__ void sfg_absorb_kernel(sfg_prog P, const sfg_verdict* V, const uint32_t* ecnt, int n,
                                             int i_base, const int32_t* scalars, int32_t* first_hit,
                                             unsigned long long* edge_delta, int32_t* key_first,
                                             unsigned long long* key_count, unsigned long long* entered_cnt,
                                             uint64_t* allocs_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // every lane stays for the warp collectives
  const int32_t stop = scalars[0];
  const bool valid = i < n;
  const int32_t g = i_base + i;
  const bool live = valid && g <= stop;
  const int lane = threadIdx.x & 31;
  const uint32_t* row = ecnt + (size_t)(valid ? i : 0) * P.n_edges;
  // per-edge first hitter / sum: warp reduce, then the CTA's warps combine in shared
  // memory and one thread per edge does the global atomics (every CTA hits the same
  // E counters: L2 atomics on a hot set, 8x fewer of them)
  __shared__ int32_t s_fh[kAbsorbEdges];
  __shared__ unsigned long long s_sum[kAbsorbEdges];
  const bool smem = P.n_edges <= kAbsorbEdges;
  if (smem)
    for (int e = threadIdx.x; e < P.n_edges; e += blockDim.x) { s_fh[e] = kNone; s_sum[e] = 0ull; }
  __syncthreads();
  for (int e = 0; e < P.n_edges; ++e) {
    const uint32_t c = valid ? row[e] : 0;
    const int32_t fh = __reduce_min_sync(0xffffffffu, c ? g : kNone);
    uint64_t s = live ? c : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (smem) {
        if (fh != kNone) atomicMin(&s_fh[e], fh);
        if (s) atomicAdd(&s_sum[e], (unsigned long long)s);
      } else {
        if (fh != kNone) atomicMin(&first_hit[e], fh);
        if (s) atomicAdd(&edge_delta[e], (unsigned long long)s);
      }
    }
  }
  __syncthreads();
  if (smem)
    for (int e = threadIdx.x; e < P.n_edges; e += blockDim.x) {
      if (s_fh[e] != kNone) atomicMin(&first_hit[e], s_fh[e]);
      if (s_sum[e]) atomicAdd(&edge_delta[e], s_sum[e]);
    }
  uint32_t ent = live ? V[i].entered : 0;
  ent = __reduce_or_sync(0xffffffffu, ent);
  if (lane == 0)
    for (uint32_t m = ent; m; m &= m - 1) atomicAdd(&entered_cnt[__ffs(m) - 1], 1ull);
  const int key = live ? V[i].key : -1;
  const unsigned mask = __ballot_sync(0xffffffffu, key >= 0);
  if (key >= 0) {
    const unsigned peers = __match_any_sync(mask, key);
    if (lane == __ffs(peers) - 1) {
      atomicMin(&key_first[key], g);
      atomicAdd(&key_count[key], (unsigned long long)__popc(peers));
    }
  }
  if (valid) allocs_out[i] = live ? (uint64_t)V[i].allocs : 0;
}

extern "C" __global__ void sfg_admit_kernel(sfg_prog P, const sfg_verdict* V, const uint32_t* ecnt,
                                            const sfg_child* ch, int n, int i_base, const int32_t* scalars,
                                            const int32_t* first_hit, const uint8_t* ghit, uint64_t* admit) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t g = i_base + i;
  uint64_t a = 0;
  if (g <= scalars[0] && V[i].status != SFG_ST_FINDING && ch[i].it != 1) {
    const uint32_t* row = ecnt + (size_t)i * P.n_edges;
    for (int e = 0; e < P.n_edges; ++e)
      if (row[e] && !ghit[e] && first_hit[e] == g) { a = 1; break; }
  }
  admit[i] = a;
}

// fold the (merged) round delta into the campaign map: saturating u64 counters
// (coverage.py:62-71), hit flags, entered-kernel mask
extern "C" __global__ void sfg_commit_kernel(int n_edges, int n_kernels, const unsigned long long* edge_delta,
                                             const unsigned long long* entered_cnt, unsigned long long* edge_total,
                                             uint8_t* ghit, uint32_t* entered) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n_edges) {
    const unsigned long long t = edge_total[e], d = edge_delta[e];
    const unsigned long long s = t + d < t ? ~0ull : t + d;
    edge_total[e] = s;
    ghit[e] = s ? 1 : 0;
  }
  if (e == 0) {
    uint32_t m = *entered;
    for (int k = 0; k < n_kernels; ++k)
      if (entered_cnt[k]) m |= 1u << k;
    *entered = m;
  }
}

// admitted children of this rank, in order, into contiguous staging rows
// (the rows every rank exchanges when a round admits)
extern "C" __global__ void sfg_select_kernel(sfg_prog P, const sfg_child* ch, const sfg_val* vals,
                                             const uint64_t* admit, const uint64_t* pos, int n, sfg_child* st_child,
                                             sfg_val* st_vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !admit[i]) return;
  const int j = (int)pos[i];
  st_child[j] = ch[i];
  for (int a = 0; a < P.n_args; ++a) st_vals[(size_t)j * P.n_args + a] = vals[(size_t)i * P.n_args + a];
}

// sizes of admitted children's pristine payloads (per input, 16-aligned per array)
extern "C" __global__ void sfg_child_bytes_kernel(sfg_prog P, const sfg_val* vals, const uint64_t* admit, int n,
                                                  uint64_t* bytes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t b = 0;
  if (!admit || admit[i]) {
    const sfg_val* v = vals + (size_t)i * P.n_args;
    for (int a = 0; a < P.n_args; ++a)
      if (v[a].kind == SFG_V_ARR) b += sfg_align16(v[a].nbytes);
  }
  bytes[i] = b;
}

// append admitted children (in `it` order) to the device corpus; emits the
// selection list and per-(selected,arg) data offsets for sfg_regen_kernel
extern "C" __global__ void sfg_compact_kernel(sfg_prog P, const sfg_child* ch, const sfg_val* vals,
                                              const uint64_t* admit, const uint64_t* pos, const uint64_t* boff,
                                              int n, int n_corpus, uint64_t corpus_bytes, sfg_entry* cmeta,
                                              sfg_val* cvals, sfg_child* cchild, int32_t* sel, uint64_t* dst_off) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (admit && !admit[i])) return;
  const int j = admit ? (int)pos[i] : i;
  const int e = n_corpus + j;
  sfg_entry m;
  m.admitted_iteration = ch[i].it;
  m.rng_seed = ch[i].rng_seed;
  m.is_seed = 0;
  m.parent = ch[i].parent;
  m.it = ch[i].it;
  cmeta[e] = m;
  cchild[e] = ch[i];
  uint64_t off = corpus_bytes + boff[i];
  for (int a = 0; a < P.n_args; ++a) {
    sfg_val v = vals[(size_t)i * P.n_args + a];
    if (v.kind == SFG_V_ARR) {
      v.data_off = off;
      dst_off[(size_t)j * P.n_args + a] = off;
      off += sfg_align16(v.nbytes);
    }
    cvals[(size_t)e * P.n_args + a] = v;
  }
  sel[j] = i;
}
