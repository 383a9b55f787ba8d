// Counter-based RNG with numpy Generator(Philox) semantics, one stream per
// fuzz input keyed on (master_seed, keybase + it).
//
// Restates the reference stream (simt_forge/rng.py:20-117), which wraps
// numpy's Philox4x64-10 bit generator and Generator draws:
//   next64       philox_next64: 4-word buffer, 256-bit counter incremented first
//   next32       philox_next32: low half first, high half cached
//   random       (next64 >> 11) * 2^-53
//   integers     Lemire bounded ints, 32-bit path below 2^32 (random_bounded_uint64_fill)
//   u64          next64
// plus the stream helpers choice / geometric_small used by the mutator.
#pragma once
#include <stdint.h>

// Philox4x64-10 of one counter block.  Out of line: every draw site (random,
// next32, integers, ...) would otherwise inline its own copy of the ten rounds,
// and the mutation kernel's code outgrew the instruction cache (ncu: 33 of 41
// cycles per issued instruction stalled on "no instruction").
struct SfgPhilox4 {
  uint64_t v0, v1, v2, v3;
};

static __device__ __noinline__ SfgPhilox4 sfg_philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                                          uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0;
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  return SfgPhilox4{c0, c1, c2, c3};
}

struct SfgStream {
  uint64_t ctr[4];
  uint64_t key0, key1;
  uint64_t buf[4];
  uint32_t pos, has32, cache32, pad;

  __device__ __forceinline__ void init(uint64_t seed, uint64_t sid) {
    ctr[0] = ctr[1] = ctr[2] = ctr[3] = 0;
    key0 = seed;
    key1 = sid;
    pos = 4;
    has32 = 0;
    cache32 = 0;
  }

  __device__ __forceinline__ void block() {
    const SfgPhilox4 o = sfg_philox4x64_10(ctr[0], ctr[1], ctr[2], ctr[3], key0, key1);
    buf[0] = o.v0; buf[1] = o.v1; buf[2] = o.v2; buf[3] = o.v3;
  }

  __device__ __forceinline__ uint64_t next64() {
    if (pos < 4) {
      // constant indices only: the buffer stays in registers (buf[pos] would put
      // the whole stream state in local memory)
      const uint64_t v = pos == 0 ? buf[0] : pos == 1 ? buf[1] : pos == 2 ? buf[2] : buf[3];
      ++pos;
      return v;
    }
    if (++ctr[0] == 0 && ++ctr[1] == 0 && ++ctr[2] == 0) ++ctr[3];
    block();
    pos = 1;
    return buf[0];
  }

  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return cache32;
    }
    const uint64_t v = next64();
    has32 = 1;
    cache32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }

  __device__ __forceinline__ double random() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }

  // numpy Generator.integers(lo, hi) for int64 dtype, hi > lo
  __device__ __forceinline__ int64_t integers(int64_t lo, int64_t hi) {
    const uint64_t rng = (uint64_t)hi - (uint64_t)lo - 1ull;
    if (rng == 0) return lo;
    if (rng <= 0xFFFFFFFFull) {
      if (rng == 0xFFFFFFFFull) return lo + (int64_t)next32();
      const uint32_t ex = (uint32_t)rng + 1u;
      uint64_t m = (uint64_t)next32() * ex;
      if ((uint32_t)m < ex) {
        const uint32_t thr = (0xFFFFFFFFu - (uint32_t)rng) % ex;
        while ((uint32_t)m < thr) m = (uint64_t)next32() * ex;
      }
      return lo + (int64_t)(m >> 32);
    }
    if (rng == ~0ull) return lo + (int64_t)next64();
    const uint64_t ex = rng + 1ull;
    uint64_t x = next64();
    uint64_t mlo = x * ex, mhi = __umul64hi(x, ex);
    if (mlo < ex) {
      const uint64_t thr = (~0ull - rng) % ex;
      while (mlo < thr) {
        x = next64();
        mlo = x * ex;
        mhi = __umul64hi(x, ex);
      }
    }
    return lo + (int64_t)mhi;
  }

  __device__ __forceinline__ int geometric_small(double p, int cap) {
    int n = 0;
    while (n < cap && random() >= p) ++n;
    return n;
  }
};
