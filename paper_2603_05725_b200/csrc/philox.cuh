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

  // numpy Generator.integers(lo, hi) for int64 dtype, 0 < hi - lo <= 2^32: the
  // 32-bit Lemire path (random_bounded_uint64_fill with rng <= 0xFFFFFFFF).  Every
  // draw of the mutator has such a range (index / count / small-constant bounds),
  // and leaving the 64-bit path out keeps each inlined draw site small (the
  // mutation kernel is instruction-fetch bound).
  __device__ __forceinline__ int64_t integers(int64_t lo, int64_t hi) {
    const uint32_t rng = (uint32_t)((uint64_t)hi - (uint64_t)lo - 1ull);
    if (rng == 0) return lo;
    if (rng == 0xFFFFFFFFu) return lo + (int64_t)next32();
    const uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)next32() * ex;
    if ((uint32_t)m < ex) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % ex;
      while ((uint32_t)m < thr) m = (uint64_t)next32() * ex;
    }
    return lo + (int64_t)(m >> 32);
  }

  // the same for any range (64-bit path above 2^32); not used by the mutator
  __device__ __forceinline__ int64_t integers64(int64_t lo, int64_t hi) {
    const uint64_t rng = (uint64_t)hi - (uint64_t)lo - 1ull;
    if (rng <= 0xFFFFFFFFull) return integers(lo, hi);
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

// Word w of a stream (block w/4 + 1, word w % 4; numpy's 256-bit counter starts
// at 0 and is incremented before every block, and 4 * 2^64 words are never
// reached).  Out of line: the rare paths of SfgWordStream / SfgWinStream.
static __device__ __noinline__ uint64_t sfg_stream_word(uint64_t key0, uint64_t key1, uint64_t w) {
  const SfgPhilox4 o = sfg_philox4x64_10(w / 4 + 1, 0, 0, 0, key0, key1);
  const uint32_t k = (uint32_t)(w & 3);
  return k == 0 ? o.v0 : k == 1 ? o.v1 : k == 2 ? o.v2 : o.v3;
}

// The block holding words b4 .. b4+3 (b4 a multiple of 4) into rows row .. row+3
// of a thread's shared-memory column (shared address scol, row pitch spitch bytes)
// when they fit (row + 4 <= cap); returns word w of it (b4 <= w < b4 + 4).
static __device__ __noinline__ uint64_t sfg_stream_refill(uint32_t scol, uint32_t spitch, uint64_t key0, uint64_t key1,
                                                          uint64_t b4, uint64_t w, uint32_t row, uint32_t cap) {
  const SfgPhilox4 o = sfg_philox4x64_10(b4 / 4 + 1, 0, 0, 0, key0, key1);
  if (row + 4 <= cap) {
    const uint32_t a = scol + row * spitch;
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(o.v0));
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a + spitch), "l"(o.v1));
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a + 2 * spitch), "l"(o.v2));
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a + 3 * spitch), "l"(o.v3));
  }
  const uint32_t k = (uint32_t)(w - b4);
  return k == 0 ? o.v0 : k == 1 ? o.v1 : k == 2 ? o.v2 : o.v3;
}

// The same draws as SfgStream, positioned by the number of 64-bit words consumed
// (w = origin + r).  Words are produced one Philox block at a time into the
// thread's column of shared memory (cap rows, a multiple of 4; later words are
// recomputed per draw), so a draw site is a compare, a shared-memory load and an
// out-of-line refill: the mutation kernel inlines ~40 draw sites and was
// instruction-fetch bound with SfgStream's register buffer and 256-bit counter
// inlined at each.
struct SfgWordStream {
  uint64_t key0, key1, origin;   // origin: word index of row 0 (a multiple of 4)
  uint32_t scol, spitch, cap, r, have, has32, cache32;

  // column: this thread's words at column[k * stride] (shared memory); a fresh
  // stream Stream(seed, sid)
  __device__ __forceinline__ void init(uint64_t* column, uint32_t stride, uint32_t cap_, uint64_t seed,
                                       uint64_t sid) {
    init_at(column, stride, cap_, seed, sid, 0, 0, 0);
  }

  // the stream after w words with the given 32-bit cache state
  __device__ __forceinline__ void init_at(uint64_t* column, uint32_t stride, uint32_t cap_, uint64_t seed,
                                          uint64_t sid, uint64_t w, uint32_t h32, uint32_t c32) {
    scol = (uint32_t)__cvta_generic_to_shared(column);
    spitch = stride * 8u;
    cap = cap_;
    key0 = seed;
    key1 = sid;
    origin = w & ~3ull;
    r = (uint32_t)(w & 3);
    have = 0;
    has32 = h32;
    cache32 = c32;
  }

  __device__ __forceinline__ uint64_t words() const { return origin + r; }

  __device__ __forceinline__ uint64_t next64() {
    uint64_t v;
    if (r < have) {
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(scol + r * spitch));
    } else {   // r == have (or past the cap): the block holding word r
      const uint32_t row = r & ~3u;
      v = sfg_stream_refill(scol, spitch, key0, key1, origin + row, origin + r, row, cap);
      if (row + 4 <= cap) have = row + 4;
    }
    ++r;
    return v;
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

  // as SfgStream::integers (0 < hi - lo <= 2^32)
  __device__ __forceinline__ int64_t integers(int64_t lo, int64_t hi) {
    const uint32_t rng = (uint32_t)((uint64_t)hi - (uint64_t)lo - 1ull);
    if (rng == 0) return lo;
    if (rng == 0xFFFFFFFFu) return lo + (int64_t)next32();
    const uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)next32() * ex;
    if ((uint32_t)m < ex) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % ex;
      while ((uint32_t)m < thr) m = (uint64_t)next32() * ex;
    }
    return lo + (int64_t)(m >> 32);
  }

  __device__ __forceinline__ int geometric_small(double p, int cap_) {
    int n = 0;
    while (n < cap_ && random() >= p) ++n;
    return n;
  }
};

// A stream positioned at an arbitrary word w whose words [wlo, wlo + nwin) sit in a
// window of shared memory shared by a warp (word k at swin + 8 * (k - wlo)); other
// words are recomputed.  The candidate walker of the sequential discipline
// (seqgen.cuh): 32 neighbouring start positions share one window.
struct SfgWinStream {
  uint64_t key0, key1, w, wlo;
  uint32_t swin, nwin, has32, cache32;

  __device__ __forceinline__ uint64_t word(uint64_t k) const {
    const uint64_t d = k - wlo;
    if (d < nwin) {
      uint64_t v;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(swin + (uint32_t)d * 8u));
      return v;
    }
    return sfg_stream_word(key0, key1, k);
  }

  __device__ __forceinline__ uint64_t next64() { return word(w++); }

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

  __device__ __forceinline__ int64_t integers(int64_t lo, int64_t hi) {
    const uint32_t rng = (uint32_t)((uint64_t)hi - (uint64_t)lo - 1ull);
    if (rng == 0) return lo;
    if (rng == 0xFFFFFFFFu) return lo + (int64_t)next32();
    const uint32_t ex = rng + 1u;
    uint64_t m = (uint64_t)next32() * ex;
    if ((uint32_t)m < ex) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % ex;
      while ((uint32_t)m < thr) m = (uint64_t)next32() * ex;
    }
    return lo + (int64_t)(m >> 32);
  }

  __device__ __forceinline__ int geometric_small(double p, int cap_) {
    int n = 0;
    while (n < cap_ && random() >= p) ++n;
    return n;
  }
};

// SfgStream state <-> words consumed.  An SfgStream that has consumed w words holds
// counter ceil(w / 4) and buffer position w - 4 * (ceil(w / 4) - 1) (4 = exhausted);
// only counter word 0 is ever non-zero.
static __device__ __forceinline__ uint64_t sfg_state_words(const SfgStream& s) {
  return s.ctr[0] == 0 ? 0ull : 4ull * (s.ctr[0] - 1ull) + s.pos;
}

static __device__ __forceinline__ void sfg_state_at(SfgStream& s, uint64_t key0, uint64_t key1, uint64_t w,
                                                    uint32_t has32, uint32_t cache32) {
  s.ctr[0] = (w + 3) / 4;
  s.ctr[1] = s.ctr[2] = s.ctr[3] = 0;
  s.key0 = key0;
  s.key1 = key1;
  s.pos = w == 0 ? 4u : (uint32_t)(w - 4 * (s.ctr[0] - 1));
  if (s.ctr[0]) {
    s.block();
  } else {
    s.buf[0] = s.buf[1] = s.buf[2] = s.buf[3] = 0;
  }
  s.has32 = has32;
  s.cache32 = cache32;
  s.pad = 0;
}

