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
