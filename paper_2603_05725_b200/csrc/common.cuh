// Small device helpers shared by the kernels.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "sfg_types.h"

#define SFG_DEV __device__ __forceinline__

SFG_DEV float sfg_f(uint32_t b) { return __uint_as_float(b); }
SFG_DEV uint32_t sfg_b(float f) { return __float_as_uint(f); }
SFG_DEV bool sfg_isnan_bits(uint32_t b) { return (b & 0x7FFFFFFFu) > 0x7F800000u; }

// NaN result of a binary32 op under the reference's host rules: the first NaN
// operand wins and is quieted; an invalid op (inf-inf, 0*inf) gives 0xFFC00000.
__device__ __noinline__ uint32_t sfg_fop_nan(uint32_t a, uint32_t b) {
  if (sfg_isnan_bits(a)) return a | 0x00400000u;
  if (sfg_isnan_bits(b)) return b | 0x00400000u;
  return 0xFFC00000u;
}

// binary32 add/sub/mul with the reference's host semantics: the value equals
// IEEE RNE (double rounding of a single f32 op is innocuous), NaN results
// follow x86-64 SSE as exhibited through ctypes.c_float (executor.py:42-44,
// 319-330).  A non-NaN result implies non-NaN operands, so the common path is
// one op and one compare.
SFG_DEV uint32_t sfg_fop(int op, uint32_t a, uint32_t b) {
  float r;
  if (op == SFG_FADD) r = __fadd_rn(sfg_f(a), sfg_f(b));
  else if (op == SFG_FSUB) r = __fsub_rn(sfg_f(a), sfg_f(b));
  else r = __fmul_rn(sfg_f(a), sfg_f(b));
  if (r == r) return sfg_b(r);
  return sfg_fop_nan(a, b);
}

// the same op where the result's NaN payload cannot be observed (jit.cu f_observers)
SFG_DEV uint32_t sfg_fop_any(int op, uint32_t a, uint32_t b) {
  if (op == SFG_FADD) return sfg_b(__fadd_rn(sfg_f(a), sfg_f(b)));
  if (op == SFG_FSUB) return sfg_b(__fsub_rn(sfg_f(a), sfg_f(b)));
  return sfg_b(__fmul_rn(sfg_f(a), sfg_f(b)));
}

SFG_DEV uint32_t sfg_quiet(uint32_t b) { return b | (sfg_isnan_bits(b) ? 0x00400000u : 0u); }

// read-only views of the device corpus (entries at round start)
struct CorpusView {
  const sfg_entry* meta;
  const sfg_val* vals;
  const uint8_t* data;
  int32_t n;        // entries at round start
  int32_t n_seeds;  // seeds form the prefix [0, n_seeds)
};

// cvt_f32_to_i32 (executor.py:51-65): NaN -> 0, saturate, round half to even
SFG_DEV uint32_t sfg_cvt_f2i(uint32_t fb) {
  const float fv = sfg_f(fb);
  if (sfg_isnan_bits(fb)) return 0u;
  if (fv >= 2147483647.0f) return 0x7FFFFFFFu;
  if (fv <= -2147483648.0f) return 0x80000000u;
  return (uint32_t)__float2int_rn(fv);
}

SFG_DEV uint64_t sfg_align16(uint64_t n) { return (n + 15ull) & ~15ull; }

// bytes an input's work region reserves for array arg value v (materialized size,
// reference PhaseRunner._materialize campaign.py:440-450)
SFG_DEV uint64_t sfg_mat_size(const sfg_val& v) {
  if (v.size_override != SFG_NO_OVERRIDE) return v.size_override > 0 ? (uint64_t)v.size_override : 0ull;
  return v.nbytes;
}

// ---------------------------------------------------------------------------
// Child payloads (mutation.py:258-357 at the data level): shared by the
// materialization kernels (mutate.cu sfg_apply / sfg_regen) and the bulk pass,
// which materializes each input's arrays itself (exec_core.cuh run_input).

static __device__ __forceinline__ uint32_t int_bits_op(uint32_t v, uint8_t kind, uint8_t sub, uint8_t byte, uint32_t mask,
                                int64_t delta) {
  if (kind == SFG_M_INT_BOUNDARY) return sub == 0 ? 0u : (sub == 1 ? 0x7FFFFFFFu : 0x80000000u);
  if (sub == 0) return v ^ ((mask & 0xFFu) << (8 * byte));      // flip
  return (uint32_t)((int64_t)(int32_t)v + delta);                // add, wraps mod 2^32
}

static __device__ __forceinline__ uint32_t float_bits_op(uint32_t b, uint8_t kind, uint8_t sub, uint8_t byte, uint32_t mask) {
  switch (kind) {                                                // mutation.py:281-306
    case SFG_M_FLOAT_SIGN: return b ^ 0x80000000u;
    case SFG_M_FLOAT_EXPONENT:
      if (sub == 0) return b | 0x7F800000u;
      if (sub == 1) return b & 0x807FFFFFu;
      return b ^ (1u << (23 + byte));
    case SFG_M_FLOAT_MANTISSA: return b ^ (mask & 0x007FFFFFu);
    case SFG_M_FLOAT_BYTE: return b ^ ((mask & 0xFFu) << (8 * byte));
    default: return sfg_fop(SFG_FADD, b, mask);                  // float_arith
  }
}

// byte p of the child's payload (p < child nbytes), given the parent's payload
static __device__ __forceinline__ uint8_t child_byte(const uint8_t* src, uint32_t src_n, const sfg_op* op,
                                              uint8_t elem, uint64_t p) {
  if (op != nullptr) {
    if (op->kind == SFG_M_ARRAY_EXTREME) {
      const uint32_t pat = elem == 1 ? (op->sub == 0 ? 0u : op->sub == 1 ? 0x7F7FFFFFu : 0xFF7FFFFFu)
                                     : (op->sub == 0 ? 0u : op->sub == 1 ? 0x7FFFFFFFu : 0x80000000u);
      return (uint8_t)(pat >> (8 * (p & 3)));
    }
    if (op->kind == SFG_M_ARRAY_ELEM && (p >> 2) == op->index) {
      const uint64_t w0 = p & ~3ull;
      uint32_t w = 0;
      for (int k = 0; k < 4; ++k) w |= (uint32_t)(w0 + k < src_n ? src[w0 + k] : 0) << (8 * k);
      if (elem == 1) w = float_bits_op(w, op->inner, op->isub, op->ibyte, op->imask);
      else w = int_bits_op(w, op->inner, op->isub, op->ibyte, op->imask, op->delta);
      return (uint8_t)(w >> (8 * (p & 3)));
    }
  }
  return p < src_n ? src[p] : 0;
}

// Write bytes [0, limit) of a child array: payload bytes where p < child nbytes,
// zeros beyond.  Lanes of a warp stride over 16-byte chunks; dst is 16-aligned.
static __device__ void emit_child(uint8_t* dst, uint64_t limit, const uint8_t* src, uint32_t src_n,
                           const sfg_val& child, const sfg_op* op, int lane, int lanes) {
  const bool extreme = op != nullptr && op->kind == SFG_M_ARRAY_EXTREME;
  const uint64_t elem_chunk =
      (op != nullptr && op->kind == SFG_M_ARRAY_ELEM) ? ((uint64_t)op->index * 4) >> 4 : ~0ull;
  const uint64_t payload = child.nbytes;
  const uint64_t copy_lim = payload < src_n ? payload : src_n;
  const bool src_al = (((uintptr_t)src) & 15) == 0;
  const uint64_t nchunks = (limit + 15) >> 4;
  // whole 16-byte chunks copied from the parent: four loads in flight per lane before
  // their stores (a lane that builds a whole input alone would otherwise wait one L2
  // round trip per chunk); the mutated element's chunk is redone below
  uint64_t c = lane;
  if (!extreme && src_al) {
    const uint64_t lim = copy_lim < limit ? copy_lim : limit;
    const uint64_t nfast = lim >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (; c + 3 * (uint64_t)lanes < nfast; c += 4 * (uint64_t)lanes) {
      const uint4 x0 = __ldg(s4 + c), x1 = __ldg(s4 + c + lanes), x2 = __ldg(s4 + c + 2 * lanes),
                  x3 = __ldg(s4 + c + 3 * lanes);
      d4[c] = x0;
      d4[c + lanes] = x1;
      d4[c + 2 * lanes] = x2;
      d4[c + 3 * lanes] = x3;
    }
    for (; c < nfast; c += lanes) d4[c] = __ldg(s4 + c);
    if (elem_chunk < nfast && elem_chunk % (uint64_t)lanes == (uint64_t)lane) {
      const uint64_t p0 = elem_chunk << 4;
      for (uint64_t p = p0; p < p0 + 16; ++p) dst[p] = child_byte(src, src_n, op, child.elem, p);
    }
  }
  for (; c < nchunks; c += lanes) {
    const uint64_t p0 = c << 4;
    if (!extreme && c != elem_chunk && src_al && p0 + 16 <= copy_lim && p0 + 16 <= limit) {
      *reinterpret_cast<uint4*>(dst + p0) = __ldg(reinterpret_cast<const uint4*>(src + p0));
      continue;
    }
    if (extreme && p0 + 16 <= payload && p0 + 16 <= limit) {
      const uint32_t pat = child.elem == 1 ? (op->sub == 0 ? 0u : op->sub == 1 ? 0x7F7FFFFFu : 0xFF7FFFFFu)
                                           : (op->sub == 0 ? 0u : op->sub == 1 ? 0x7FFFFFFFu : 0x80000000u);
      *reinterpret_cast<uint4*>(dst + p0) = make_uint4(pat, pat, pat, pat);
      continue;
    }
    if (p0 >= payload && p0 + 16 <= limit) {
      *reinterpret_cast<uint4*>(dst + p0) = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint64_t pe = p0 + 16 < limit ? p0 + 16 : limit;
    for (uint64_t p = p0; p < pe; ++p) dst[p] = p < payload ? child_byte(src, src_n, op, child.elem, p) : 0;
  }
}
