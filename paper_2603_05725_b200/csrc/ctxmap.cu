// K4b: context-sensitive hashed coverage map (BASELINE.json configs[2]; the
// north star's "(calling context, edge) hashed into bitmaps, merged with a
// warp-ballot novelty pass and an OR/MAX all-reduce across GPUs").
//
// A derived view beside the exact per-edge map the reference keeps
// (coverage.py:40-94): novelty and admission stay on exact dense edge ids
// (collisions here must not change admissions).
//
// Map: 2^bits one-byte slots (bits = 24 -> 16 MiB), 0 = unseen, 1 = seen.
// A live input that hit edge e c times sets slot
//     fmix64(edge_ctx[e] ^ bucket(c) * golden) & (2^bits - 1)
// where edge_ctx[e] (host, lowering.ctx_edge_hashes) hashes the launch-chain
// context of the edge's kernel with (kernel, src, dst), and bucket() is the
// AFL hit-count class (1, 2, 3, 4-7, 8-15, 16-31, 32-127, 128+).  Byte flags
// make the cross-GPU merge an exact MAX all-reduce (NCCL has no OR).
#include "common.cuh"

namespace {
SFG_DEV uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

SFG_DEV uint32_t hit_bucket(uint32_t c) {
  if (c <= 3) return c;
  if (c < 8) return 4;
  if (c < 16) return 5;
  if (c < 32) return 6;
  if (c < 128) return 7;
  return 8;
}
}  // namespace

// one thread per (input, edge); warp-aggregated test-and-set on the containing
// 32-bit word; new_slots[0] += slots this launch turned on
extern "C" __global__ void sfg_ctxmap_kernel(int n, int n_edges, int i_base, const uint32_t* ecnt,
                                             const int32_t* scalars, const uint64_t* edge_ctx, uint32_t* map_words,
                                             uint64_t mask, unsigned long long* new_slots) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n * n_edges;
  const int lane = threadIdx.x & 31;
  bool act = false;
  uint64_t slot = 0;
  if (t < total) {
    const int i = (int)(t / n_edges), e = (int)(t % n_edges);
    const uint32_t c = ecnt[t];
    if (c && i_base + i <= scalars[0]) {
      act = true;
      slot = fmix64(edge_ctx[e] ^ ((uint64_t)hit_bucket(c) * 0x9E3779B97F4A7C15ull)) & mask;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, act);
  unsigned fresh = 0;
  if (act) {
    const unsigned peers = __match_any_sync(m, slot);
    if (lane == __ffs(peers) - 1) {
      const uint32_t bit = 1u << (8 * (slot & 3));
      const uint32_t old = atomicOr(&map_words[slot >> 2], bit);
      fresh = (old & bit) ? 0u : 1u;
    }
  }
  fresh = __reduce_add_sync(0xffffffffu, fresh);
  if (lane == 0 && fresh) atomicAdd(new_slots, (unsigned long long)fresh);
}
