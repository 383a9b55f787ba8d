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
                                                 int* sig) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  const int b = active ? sig_bucket(P, vals + (size_t)i * P.n_args, mask) : 0;
  if (active) sig[i] = b;
  warp_agg_add(hist, b, active);
}

// exclusive scan of the kOrderBuckets counts by one small CTA (128 threads x 32
// buckets): it must find room on SMs busy with other rounds' long inputs
extern "C" __global__ void __launch_bounds__(128) sfg_order_scan_kernel(int* hist) {
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
}

extern "C" __global__ void sfg_order_scatter_kernel(int n, const int* sig, int* offs, int32_t* order) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  const int b = active ? sig[i] : 0;
  const int pos = warp_agg_add(offs, b, active);
  if (active) order[pos] = i;
}
