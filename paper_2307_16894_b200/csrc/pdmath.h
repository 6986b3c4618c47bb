// Portable table-driven fp64 exp / log (host and device, identical
// operation sequence with explicit fma()).
//
// Why: the material's FD tangent divides ulp-level differences of P by 2h
// (~2e-7), so the CPU<->GPU tangent gap is set by how often the device
// exp/log round differently from the host's.  libdevice
// exp/log are ~1 ulp; these are ~0.5 + 2^-6 ulp (nearly correctly rounded,
// like glibc's), and the same source compiled for the host reproduces the
// device results bit for bit (tests: GPU == oracle built with this libm).
// They are also cheaper: exp ~12 DP instructions (libdevice 16), log ~23
// (libdevice 29).
//
//   exp(x) = 2^(k/256) e^r,  k = round(256 x / ln 2), |r| <= ln2/512,
//            e^r - 1 by its degree-5 Taylor polynomial (truncation < 1e-20),
//            2^(j/256) as hi + lo from a 256-entry table.
//   log(x) = e ln2 - log(invc) + log1p(r),  r = z invc - 1 EXACT (invc ~ 1/c
//            with 8 significant bits, c the centre of one of 128 mantissa
//            intervals; invc = 1 on the two intervals touching 1 so x ~ 1
//            never cancels), |r| < 2^-7, log1p by its degree-9 Taylor
//            polynomial (truncation < 2^-73 relative),
//            hi/lo bookkeeping with two Fast2Sum steps.
// Inputs outside the fast range (|x| >= 700 for exp; x <= 0, subnormal, inf,
// nan for log) fall back to the platform function.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define PDM_HD __device__ __forceinline__
#define PDM_TABLE static __device__ const
#define PDM_KTAB static __constant__
#else
#define PDM_HD inline
#define PDM_TABLE static const
#define PDM_KTAB static const
#endif

#include "pdmath_tables.h"

// Reduction and polynomial constants.  On the device they sit in the
// constant bank, so the FP64 instructions take them as c[][] operands; a
// double literal whose low word is nonzero costs two UMOVs per use instead
// (about 9 % of the material kernel's issued instructions).
PDM_KTAB double pdm_k[12] = {
    PDM_EXP_INVLN2N, PDM_EXP_LN2N_HI, PDM_EXP_LN2N_LO,  // exp reduction
    1.0 / 120.0,     1.0 / 24.0,      1.0 / 6.0,        // exp Taylor c5, c4, c3
    1.0 / 9.0,       1.0 / 7.0,       1.0 / 5.0,        // log1p Taylor
    1.0 / 3.0,       PDM_LN2_HI,      PDM_LN2_LO,
};

namespace pdm {

enum {
  kInvLn2N = 0, kLn2NHi, kLn2NLo, kC5, kC4, kC3, kL9, kL7, kL5, kL3, kLn2Hi, kLn2Lo
};

PDM_HD double tab(const double* t, int i) {
#ifdef __CUDA_ARCH__
  return __ldg(t + i);
#else
  return t[i];
#endif
}

PDM_HD uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, sizeof(u));
  return u;
#endif
}

PDM_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  std::memcpy(&x, &u, sizeof(x));
  return x;
#endif
}

PDM_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return fma(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

PDM_HD bool exp_fast_ok(double x) { return x > -700.0 && x < 700.0; }

// Fast path only (callers check exp_fast_ok); on an out-of-range input it
// returns garbage without faulting (saturating conversions, masked index).
PDM_HD double exp_core(double x) {
  const double shift = 0x1.8p52;
  double kd = fma_(x, pdm_k[kInvLn2N], shift);
  kd = kd - shift;                       // round(256 x / ln2), exact integer
  double r = fma_(kd, -pdm_k[kLn2NHi], x);
  r = fma_(kd, -pdm_k[kLn2NLo], r);
  const int k = (int)kd;
  const int j = k & 255;
  const int e = (k - j) / 256;           // floor(k / 256)
  const double r2 = r * r;
  const double poly = fma_(fma_(fma_(r, pdm_k[kC5], pdm_k[kC4]), r, pdm_k[kC3]), r, 0.5);
  const double p = fma_(r2, poly, r);    // e^r - 1
  const double th = tab(pdm_exp_tab, 2 * j), tl = tab(pdm_exp_tab, 2 * j + 1);
  const double res = th + fma_(th, p, tl);
  return res * from_bits((uint64_t)(e + 1023) << 52);  // exact power-of-two scale
}

PDM_HD double exp(double x) {
  if (!exp_fast_ok(x)) {
#ifdef __CUDA_ARCH__
    return ::exp(x);
#else
    return std::exp(x);
#endif
  }
  return exp_core(x);
}

// x > 0 normal and finite (otherwise: x <= 0, subnormal, inf, nan; a set
// sign bit makes top >= 0x800)
PDM_HD bool log_fast_ok(double x) { return (uint32_t)(bits(x) >> 52) - 1u < 0x7feu; }

// Fast path only (callers check log_fast_ok); garbage but no fault otherwise.
PDM_HD double log_core(double x) {
  const uint64_t ix = bits(x);
  const uint32_t top = (uint32_t)(ix >> 52);
  int e = (int)top - 1023;
  const int i = (int)((ix >> 45) & 127);
  uint64_t mb = (ix & 0x000fffffffffffffull) | 0x3ff0000000000000ull;  // m in [1, 2)
  if (i >= PDM_LOG_HALF_FROM) {  // m >= ~sqrt 2: use m / 2 in [0.707, 1)
    mb -= 0x0010000000000000ull;
    e += 1;
  }
  const double z = from_bits(mb);
  const double invc = tab(pdm_log_tab, 3 * i);
  const double lhi = tab(pdm_log_tab, 3 * i + 1), llo = tab(pdm_log_tab, 3 * i + 2);
  const double r = fma_(z, invc, -1.0);
  const double r2 = r * r;
  double q = fma_(r, pdm_k[kL9], -0.125);
  q = fma_(q, r, pdm_k[kL7]);
  q = fma_(q, r, -pdm_k[kC3]);           // -1/6
  q = fma_(q, r, pdm_k[kL5]);
  q = fma_(q, r, -0.25);
  q = fma_(q, r, pdm_k[kL3]);
  q = fma_(q, r, -0.5);
  q = r2 * q;                            // log1p(r) - r
  const double ed = (double)e;
  const double t = ed * pdm_k[kLn2Hi];      // exact (PDM_LN2_HI has 41 significant bits)
  const double s = t + lhi;
  const double s_err = (t - s) + lhi;    // Fast2Sum, |t| >= |lhi| or t == 0
  const double hh = s + r;
  const double h_err = (s - hh) + r;     // Fast2Sum, |s| >= |r| or s == 0
  const double lo = ((fma_(ed, pdm_k[kLn2Lo], s_err) + llo) + h_err) + q;
  return hh + lo;
}

PDM_HD double log(double x) {
  if (!log_fast_ok(x)) {
#ifdef __CUDA_ARCH__
    return ::log(x);
#else
    return std::log(x);
#endif
  }
  return log_core(x);
}

// Two independent evaluations with one range branch: both fast paths are
// straight-line code the scheduler can interleave (instruction-level
// parallelism for the FP64 pipe); results are exactly exp(x0), exp(x1).
PDM_HD void exp_pair(double x0, double x1, double& r0, double& r1) {
#ifndef __CUDA_ARCH__
  r0 = pdm::exp(x0);  // host: no speculative fast path (int conversion UB)
  r1 = pdm::exp(x1);
  return;
#endif
  r0 = exp_core(x0);
  r1 = exp_core(x1);
  if (!(exp_fast_ok(x0) && exp_fast_ok(x1))) {
    r0 = pdm::exp(x0);
    r1 = pdm::exp(x1);
  }
}

PDM_HD void log_pair(double x0, double x1, double& r0, double& r1) {
#ifndef __CUDA_ARCH__
  r0 = pdm::log(x0);
  r1 = pdm::log(x1);
  return;
#endif
  r0 = log_core(x0);
  r1 = log_core(x1);
  if (!(log_fast_ok(x0) && log_fast_ok(x1))) {
    r0 = pdm::log(x0);
    r1 = pdm::log(x1);
  }
}

}  // namespace pdm
