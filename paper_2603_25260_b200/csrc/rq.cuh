// rq.cuh — the fixed-point requantisation of Eq.14 (reading Q18: PReLU = sign-selected
// multiplier), used by every int8-producing epilogue of the CUDA path.
//
//   rq(x) = clip( floor((x * m + 2^(r-1)) / 2^r), -128, 127 ),  m = x >= 0 ? m_pos : m_neg
//
// Generic form: one 64-bit product and shift.  Fast form (RQ::fast, set at model load
// when 1 <= r <= 32 and m_pos, m_neg < 2^r): multiplying numerator and denominator of
// the floor by 2^(32-r) gives, with M = m * 2^(32-r) < 2^32 and y = |x| < 2^31,
//   x >= 0:  rq(x) =  hi32(y * M + 2^31)
//   x <  0:  rq(x) = -hi32(y * M + 2^31 - 2^(32-r))      (floor of a negative = -ceil)
// one IMAD.WIDE.U32 instead of the 64-bit multiply/add/shift sequence; y*M + A < 2^63
// so nothing overflows and the result is bit-identical to the generic form.
// Signed form (RQ::fast_s, when additionally m_pos, m_neg < 2^(r-1), so M < 2^31 fits a
// signed 32-bit operand): rq(x) = clip( (int64(x) * M + 2^31) >> 32 ) for either sign
// (the arithmetic shift is the floor), |x * M| < 2^62: one IMAD.WIDE, no sign fix-up.
#pragma once
#include "pcc_internal.cuh"

namespace pcc {

__host__ __device__ inline void rq_prepare(RQ& q) {
  q.fast = q.fast_s = 0;
  q.Mp = q.Mn = q.Ap = q.An = 0;
  q.Sp = q.Sn = 0;
  if (q.r >= 1 && q.r <= 32 && (int64_t(q.mp) >> q.r) == 0 && (int64_t(q.mn) >> q.r) == 0) {
    q.fast = 1;
    q.Mp = uint32_t(uint64_t(q.mp) << (32 - q.r));
    q.Mn = uint32_t(uint64_t(q.mn) << (32 - q.r));
    q.Ap = 0x80000000u;
    q.An = 0x80000000u - uint32_t(uint64_t(1) << (32 - q.r));
    if ((int64_t(q.mp) >> (q.r - 1)) == 0 && (int64_t(q.mn) >> (q.r - 1)) == 0) {
      q.fast_s = 1;
      q.Sp = int32_t(q.Mp);
      q.Sn = int32_t(q.Mn);
    }
  }
}

// signed form, unclamped (callers saturate, e.g. with cvt.pack.sat): valid iff q.fast_s
__device__ __forceinline__ int32_t rq_s(int32_t x, const RQ& q) {
  const int64_t p = int64_t(x) * int64_t(x < 0 ? q.Sn : q.Sp) + (int64_t(1) << 31);
  return int32_t(p >> 32);
}

// four int32 -> four saturated int8 packed little-endian (a lowest)
__device__ __forceinline__ uint32_t pack_sat4(int32_t a, int32_t b, int32_t c, int32_t d) {
  uint32_t hi, out;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(out) : "r"(b), "r"(a), "r"(hi));
  return out;
}

__device__ __forceinline__ int32_t rq8_generic(int32_t x, const RQ& q) {
  int64_t v = int64_t(x) * int64_t(x >= 0 ? q.mp : q.mn);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  return int32_t(v < -128 ? -128 : (v > 127 ? 127 : v));
}

__device__ __forceinline__ int32_t rq8(int32_t x, const RQ& q) {
  if (!q.fast) return rq8_generic(x, q);
  const bool neg = x < 0;
  const uint32_t y = neg ? 0u - uint32_t(x) : uint32_t(x);
  const uint64_t p = uint64_t(y) * (neg ? q.Mn : q.Mp) + (neg ? q.An : q.Ap);
  const int32_t h = int32_t(uint32_t(p >> 32));
  return neg ? max(-h, -128) : min(h, 127);
}

}  // namespace pcc
