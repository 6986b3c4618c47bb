// The host's glibc exp/log, restated for the device (and the host, for the
// bitwise checks): the material's default libm.
//
// The reference evaluates std::exp / std::log (material.cpp:135-150) with
// glibc, whose x86-64 IFUNCs select the FMA builds of sysdeps/ieee754/dbl-64
// e_exp.c / e_log.c on an AVX2+FMA host (glibc 2.39, Ubuntu 24.04; the
// implementation the oracle and the reference execute here and on the GPU
// box).  Those are table-driven ~0.51-ulp algorithms:
//
//   exp(x) = 2^(k/128) (1 + tail_k + r + C2 r^2 + ... + C5 r^5),
//            k = round(128 x / ln2), r = x - k ln2/128 (hi/lo split),
//   log(x) = k ln2 + log(c_i) + poly(z invc_i - 1)  with x = 2^k z,
//            or a degree-12 polynomial in r = x - 1 with a hi/lo split of
//            the r^2/2 term when x is within [1 - 2^-4, 1 + 0x1.09p-4).
//
// Every operation below is the one the compiled FMA variant executes, in its
// order, with fma() exactly where the machine code has a vfmadd (read off
// `objdump -d` of the IFUNC targets; DESIGN.md §3 lists the mapping).  The
// data (__exp_data / __log_data) is lifted from libm.so.6 by
// tools/gen_gmath_tables.py into gmath_tables.h.  Result: gm::exp / gm::log
// equal glibc's bit for bit (tests/test_gmath.py: >= 2^30 arguments per
// function on the host; tests/test_gpu_gmath.py on the device), so the
// device material reproduces the glibc oracle bit for bit.
//
// The material kernels use the pair forms: both fast paths of two calls
// are straight-line code (the near-1 and general log paths are both
// evaluated and one selected), with one rare-path branch for arguments
// outside them (|x| >= 512 and nan for exp; zero, negative, subnormal, inf,
// nan for log).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define GM_HD __device__ __forceinline__
#define GM_NOINLINE static __device__ __noinline__
#define GM_TABLE static __device__ const
#define GM_KTAB static __constant__
#else
#define GM_HD inline
#define GM_NOINLINE inline
#define GM_TABLE static const
#define GM_KTAB static const
#endif

#include "gmath_tables.h"

GM_KTAB double gm_ek[8] = {GM_EXP_K_INIT};
GM_KTAB double gm_lk[18] = {GM_LOG_K_INIT};

namespace gm {

enum { kInvLn2N = 0, kShift, kNegLn2hiN, kNegLn2loN, kC2, kC3, kC4, kC5 };
enum { kLn2hi = 0, kLn2lo, kA0, kA1, kA2, kA3, kA4, kB0, kB1, kB2, kB3, kB4, kB5, kB6, kB7, kB8, kB9,
       kB10 };

GM_HD uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, sizeof(u));
  return u;
#endif
}

GM_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  std::memcpy(&x, &u, sizeof(x));
  return x;
#endif
}

GM_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return fma(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// Table pairs (exp: tail, scale bits; log: invc, logc) as one 16-byte load.
GM_HD void etab2(int k, uint64_t& tail, uint64_t& sb) {
#ifdef __CUDA_ARCH__
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(gm_exp_tab) + k);
  tail = v.x;
  sb = v.y;
#else
  tail = gm_exp_tab[2 * k];
  sb = gm_exp_tab[2 * k + 1];
#endif
}

GM_HD void ltab2(int i, double& invc, double& logc) {
#ifdef __CUDA_ARCH__
  const double2 v = __ldg(reinterpret_cast<const double2*>(gm_log_tab) + i);
  invc = v.x;
  logc = v.y;
#else
  invc = gm_log_tab[2 * i];
  logc = gm_log_tab[2 * i + 1];
#endif
}

// |x| in [2^-54, 512): the main path needs no special case.
GM_HD bool exp_main_ok(double x) {
  const uint32_t abstop = (uint32_t)(bits(x) >> 52) & 0x7ffu;
  return abstop - 0x3c9u < 0x3fu;
}

// Main path up to the final scale (e_exp.c __exp, FMA build).  kd's integer
// bits give the table index and the exponent; only the low 19 bits of ki
// reach the result (ki << 45), so a 32-bit view suffices.
GM_HD void exp_tmp(double x, double& tmp, uint64_t& sbits, uint32_t& ki_lo) {
  double kd = fma_(x, gm_ek[kInvLn2N], gm_ek[kShift]);
  const uint64_t ki = bits(kd);
  kd = kd - gm_ek[kShift];
  double r = fma_(kd, gm_ek[kNegLn2hiN], x);
  r = fma_(kd, gm_ek[kNegLn2loN], r);
  uint64_t tb, sb;
  etab2((int)(ki & 127u), tb, sb);
  const double tail = from_bits(tb);
  sbits = sb + (ki << 45);
  ki_lo = (uint32_t)ki;
  const double r2 = r * r;
  const double t = r + tail;
  const double p23 = fma_(r, gm_ek[kC3], gm_ek[kC2]);
  const double p45 = fma_(r, gm_ek[kC5], gm_ek[kC4]);
  const double a = fma_(p23, r2, t);
  const double r4 = r2 * r2;
  tmp = fma_(r4, p45, a);
}

GM_HD double exp_core(double x) {
  double tmp;
  uint64_t sbits;
  uint32_t ki;
  exp_tmp(x, tmp, sbits, ki);
  const double scale = from_bits(sbits);
  return fma_(scale, tmp, scale);
}

// Everything outside the main range: |x| < 2^-54, |x| >= 512 (scaled
// "specialcase"), infinities and nan (e_exp.c's early exits, __math_oflow /
// __math_uflow values).
GM_NOINLINE double exp_rare(double x) {
  const uint64_t ix = bits(x);
  const uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop < 0x3c9u) return 1.0 + x;
  if (abstop >= 0x409u) {
    if (ix == 0xfff0000000000000ull) return 0.0;
    if (abstop == 0x7ffu) return 1.0 + x;
    return (ix >> 63) ? 0.0 : from_bits(0x7ff0000000000000ull);
  }
  double tmp;
  uint64_t sbits;
  uint32_t ki;
  exp_tmp(x, tmp, sbits, ki);
  if ((ki & 0x80000000u) == 0) {  // k > 0: the scale's exponent may overflow
    sbits -= 1009ull << 52;
    const double scale = from_bits(sbits);
    return fma_(scale, tmp, scale) * 0x1p1009;
  }
  sbits += 1022ull << 52;  // k < 0: subnormal range
  const double scale = from_bits(sbits);
  const double st = tmp * scale;
  double y = scale + st;
  if (1.0 > y) {
    const double hi = y + 1.0;
    double lo = (scale - y) + st;
    lo = ((1.0 - hi) + y) + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return y * 0x1p-1022;
}

// |x| < 512: the main path.  Below 2^-54 glibc returns 1 + x instead, and
// exp_core gives the same bits there: kd = Shift exactly, so k = 0, r = x,
// tail = 0, scale = 1, |tmp| = |x| (1 + tiny) < 2^-54 and RN(1 + tmp) =
// RN(1 + x) = 1 (zeros and subnormals included; tests/test_gmath.py checks
// exp_core against glibc over the whole tiny range).  So the elastic branch's
// exp(+0) needs no special path.
GM_HD bool exp_fast_ok(double x) { return ((uint32_t)(bits(x) >> 52) & 0x7ffu) < 0x408u; }

GM_HD double exp_fast(double x) { return exp_core(x); }

GM_HD double exp(double x) { return exp_main_ok(x) ? exp_core(x) : exp_rare(x); }

// ---- log
constexpr uint64_t kLogLo = 0x3fee000000000000ull;  // asuint64(1 - 0x1p-4)
constexpr uint64_t kLogHi = 0x3ff1090000000000ull;  // asuint64(1 + 0x1.09p-4)
constexpr uint64_t kLogOff = 0x3fe6000000000000ull;

// Normal, positive, finite (the near-1 and general paths).
GM_HD bool log_main_ok(double x) {
  const uint32_t top = (uint32_t)(bits(x) >> 48);
  return top - 0x0010u < 0x7ff0u - 0x0010u;
}

GM_HD bool log_near1(uint64_t ix) { return ix - kLogLo < kLogHi - kLogLo; }

// General path for a normal positive ix (e_log.c __log, FMA build).
GM_HD double log_general(uint64_t ix) {
  const uint64_t tmp = ix - kLogOff;
  const int i = (int)((tmp >> 45) & 127u);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  double invc, logc;
  ltab2(i, invc, logc);
  const double z = from_bits(iz);
  const double kd = (double)k;
  const double w = fma_(kd, gm_lk[kLn2hi], logc);
  const double r = fma_(z, invc, -1.0);
  const double p12 = fma_(r, gm_lk[kA2], gm_lk[kA1]);
  const double hi = r + w;
  const double r2 = r * r;
  const double lo = fma_(kd, gm_lk[kLn2lo], (w - hi) + r);
  const double r3 = r * r2;
  const double p34 = fma_(r, gm_lk[kA4], gm_lk[kA3]);
  const double lo2 = fma_(r2, gm_lk[kA0], lo);
  const double q = fma_(p34, r2, p12);
  const double y = fma_(r3, q, lo2);
  return y + hi;
}

// Near-1 path: x in [1 - 2^-4, 1 + 0x1.09p-4).
GM_HD double log_near(double x) {
  const double r = x - 1.0;
  const double b12 = fma_(r, gm_lk[kB2], gm_lk[kB1]);
  const double b45 = fma_(r, gm_lk[kB5], gm_lk[kB4]);
  const double b78 = fma_(r, gm_lk[kB8], gm_lk[kB7]);
  const double r2 = r * r;
  const double b13 = fma_(r2, gm_lk[kB3], b12);
  const double b46 = fma_(r2, gm_lk[kB6], b45);
  const double r3 = r * r2;
  const double b79 = fma_(r2, gm_lk[kB9], b78);
  const double b710 = fma_(r3, gm_lk[kB10], b79);
  const double u = fma_(b710, r3, b46);
  const double poly = fma_(u, r3, b13);
  const double t = fma_(r, 0x1p27, r);
  const double rhi = fma_(-0x1p27, r, t);
  const double rhi2 = rhi * rhi;
  const double rlo = r - rhi;
  const double hi = fma_(rhi2, gm_lk[kB0], r);
  const double d = r - hi;
  const double s = r + rhi;
  double lo = fma_(rhi2, gm_lk[kB0], d);
  const double m = gm_lk[kB0] * rlo;
  lo = fma_(m, s, lo);
  const double y = fma_(poly, r3, lo);
  return hi + y;
}

// Both paths evaluated, one selected (branch-free; x normal positive).
// glibc returns +0 for x == 1 explicitly (the sign of zero under downward
// rounding); under round-to-nearest the near-1 path yields +0 there too
// (r = +0 and every term is a signed zero that sums to +0), so no select.
GM_HD double log_core(double x) {
  const uint64_t ix = bits(x);
  const double g = log_general(ix);
  const double n = log_near(x);
  return log_near1(ix) ? n : g;
}

// Zero, negative, subnormal, inf, nan (e_log.c's special-case block).
GM_NOINLINE double log_rare(double x) {
  uint64_t ix = bits(x);
  if (log_near1(ix)) return ix == 0x3ff0000000000000ull ? 0.0 : log_near(x);
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if (ix * 2 == 0) return -from_bits(0x7ff0000000000000ull);  // -inf (divzero)
    if (ix == 0x7ff0000000000000ull) return x;                   // log(inf) == inf
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) {
      const double z = x - x;
      return z / z;  // nan (invalid)
    }
    ix = bits(x * 0x1p52) - (52ull << 52);  // subnormal: normalise
  }
  return log_general(ix);
}

GM_HD double log(double x) {
  if (!log_main_ok(x)) return log_rare(x);
  const uint64_t ix = bits(x);
  if (log_near1(ix)) return ix == 0x3ff0000000000000ull ? 0.0 : log_near(x);
  return log_general(ix);
}

// Pair forms for the material kernels: two straight-line evaluations and a
// single rare-path branch.  Results are exactly exp(x0), exp(x1) / log(..).
GM_HD void exp_pair(double x0, double x1, double& r0, double& r1) {
#ifndef __CUDA_ARCH__
  r0 = gm::exp(x0);
  r1 = gm::exp(x1);
#else
  r0 = exp_fast(x0);
  r1 = exp_fast(x1);
  if (!(exp_fast_ok(x0) && exp_fast_ok(x1))) {
    r0 = gm::exp(x0);
    r1 = gm::exp(x1);
  }
#endif
}

// Device: both paths in every lane, one selected.  With -DGM_WARP_LOG the
// near-1 path (24 FP64 instructions, needed for a minority of arguments but
// by almost every warp) runs once per warp on the warp's near-1 arguments
// packed into consecutive lanes (ballot ranks; fetched and returned by
// shuffles) — bit-identical, but measured slower in the material kernel
// (1.205 against 1.09 ms per config-1 step: the shuffles and ranks sit on
// the critical path of every evaluation), so it is off by default.
GM_HD void log_pair(double x0, double x1, double& r0, double& r1) {
#ifndef __CUDA_ARCH__
  r0 = gm::log(x0);
  r1 = gm::log(x1);
#elif !defined(GM_WARP_LOG)
  r0 = log_core(x0);
  r1 = log_core(x1);
  if (!(log_main_ok(x0) && log_main_ok(x1))) {
    r0 = gm::log(x0);
    r1 = gm::log(x1);
  }
#else
  const uint64_t i0 = bits(x0), i1 = bits(x1);
  r0 = log_general(i0);
  r1 = log_general(i1);
  const bool n0 = log_near1(i0), n1 = log_near1(i1);
  const unsigned act = __activemask();
  const unsigned b0 = __ballot_sync(act, n0), b1 = __ballot_sync(act, n1);
  if (b0 | b1) {
    const int c0 = __popc(b0), c = c0 + __popc(b1);
    const int nact = __popc(act);
    if (c <= nact) {
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      const bool full = act == 0xffffffffu;
      const int rank = __popc(act & lt);
      const int lane = __popc(lt);
      int src = lane;
      bool second = false;
      if (rank < c) {  // this lane evaluates slot `rank` of the packed list
        second = rank >= c0;
        src = (int)__fns(second ? b1 : b0, 0, (second ? rank - c0 : rank) + 1);
      }
      const double a0 = __shfl_sync(act, x0, src), a1 = __shfl_sync(act, x1, src);
      const double v = log_near(second ? a1 : a0);
      const int s0 = __popc(b0 & lt), s1 = c0 + __popc(b1 & lt);
      const int h0 = full ? s0 : (int)__fns(act, 0, s0 + 1);
      const int h1 = full ? s1 : (int)__fns(act, 0, s1 + 1);
      const double v0 = __shfl_sync(act, v, h0 & 31), v1 = __shfl_sync(act, v, h1 & 31);
      r0 = n0 ? v0 : r0;
      r1 = n1 ? v1 : r1;
    } else {
      const double v0 = log_near(x0), v1 = log_near(x1);
      r0 = n0 ? v0 : r0;
      r1 = n1 ? v1 : r1;
    }
  }
  if (!(log_main_ok(x0) && log_main_ok(x1))) {
    r0 = gm::log(x0);
    r1 = gm::log(x1);
  }
#endif
}

}  // namespace gm
