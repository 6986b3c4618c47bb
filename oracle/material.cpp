// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/src/material.cpp:10-181.
#include "oracle.hpp"

#include <algorithm>

// The reference calls glibc's std::log / std::exp.  Built with -DORC_PDMATH
// (liboracle_pdm.so) the oracle uses the device's portable exp/log instead:
// that variant isolates the libm from the algorithm (GPU == oracle bit for
// bit), while the default build is the faithful glibc restatement.
#ifdef ORC_PDMATH
#include "../paper_2307_16894_b200/csrc/pdmath.h"
#define ORC_LOG pdm::log
#define ORC_EXP pdm::exp
#else
#define ORC_LOG std::log
#define ORC_EXP std::exp
#endif

namespace orc {

namespace {

// material.cpp:41-55 (eig_sym2): closed-form symmetric 2x2 eigenpairs.
struct Eig2 {
  double l1 = 0, l2 = 0;
  double v1[2] = {1, 0}, v2[2] = {0, 1};
};

Eig2 eig_sym2(const Mat2& c) {
  Eig2 e;
  const double tr = c(0, 0) + c(1, 1);
  const double hd = 0.5 * (c(0, 0) - c(1, 1));
  const double off = 0.5 * (c(0, 1) + c(1, 0));
  const double d = std::sqrt(hd * hd + off * off);
  e.l1 = 0.5 * tr + d;
  e.l2 = 0.5 * tr - d;
  if (d <= 1e-14 * (std::abs(tr) + 1.0)) return e;  // repeated root: axis frame
  double vx = off, vy = e.l1 - c(0, 0);
  if (vx * vx + vy * vy < 1e-30 * d * d) {
    vx = e.l1 - c(1, 1);
    vy = off;
  }
  const double nrm = std::sqrt(vx * vx + vy * vy);  // Eigen normalized(): v / sqrt(|v|^2)
  e.v1[0] = vx / nrm;
  e.v1[1] = vy / nrm;
  e.v2[0] = -e.v1[1];
  e.v2[1] = e.v1[0];
  return e;
}

}  // namespace

// material.cpp:80-118.  Components [xx, yy, zz, xy].  The 4x4 consistent
// tangent (:109-114) is never consumed by the finite-strain path and is
// omitted here.
SmallResult small_strain_update(const PlasticityParams& p, const double eps_p0[4], double xi0,
                                const double eps[4], double eps_p1[4], double* xi1) {
  const double la = p.lambda(), mu = p.mu();
  SmallResult r;
  double ee[4];
  for (int k = 0; k < 4; ++k) ee[k] = eps[k] - eps_p0[k];
  const double tr = ee[0] + ee[1] + ee[2];
  double st[4] = {la * tr + 2 * mu * ee[0], la * tr + 2 * mu * ee[1], la * tr + 2 * mu * ee[2],
                  2 * mu * ee[3]};
  const double pm = (st[0] + st[1] + st[2]) / 3.0;  // deviator(), :15-17
  const double dev[4] = {st[0] - pm, st[1] - pm, st[2] - pm, st[3]};
  // sym_dot(), :10-12
  const double nd = std::sqrt(dev[0] * dev[0] + dev[1] * dev[1] + dev[2] * dev[2] +
                              2.0 * dev[3] * dev[3]);
  r.q_trial = std::sqrt(1.5) * nd;
  r.f_trial = r.q_trial - (p.sigma_y0 + p.H * xi0);
  for (int k = 0; k < 4; ++k) eps_p1[k] = eps_p0[k];
  double xn = xi0;
  if (r.f_trial <= 0.0) {
    for (int k = 0; k < 4; ++k) r.sigma[k] = st[k];
    r.mises = r.q_trial;
  } else {
    r.dgamma = r.f_trial / (3 * mu + p.H);
    const double c = 1.5 / r.q_trial;
    const double s = 2 * mu * r.dgamma;
    for (int k = 0; k < 4; ++k) {
      const double rk = c * dev[k];  // flow direction
      r.sigma[k] = st[k] - s * rk;
      eps_p1[k] += r.dgamma * rk;
    }
    xn += r.dgamma;
    r.mises = r.q_trial - 3 * mu * r.dgamma;
  }
  if (xi1) *xi1 = xn;
  return r;
}

// material.cpp:120-162.
LargeResult large_strain_update(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                                PlasticState* s1) {
  const Mat2 fp0_inv = inverse(s0.Fp);
  const Mat2 fe = mul(F, fp0_inv);
  const Mat2 c = mul(transpose(fe), fe);
  const double czz = 1.0 / (s0.Fp_zz * s0.Fp_zz);
  const Eig2 eg = eig_sym2(c);
  if (eg.l2 <= 0.0 || czz <= 0.0)
    throw SolveError("plasticity update hit a non-positive elastic stretch (det F = " +
                     std::to_string(det(F)) + ")");

  const double eps_tr[4] = {0.5 * ORC_LOG(eg.l1), 0.5 * ORC_LOG(eg.l2), 0.5 * ORC_LOG(czz), 0.0};
  // Quirk replicated: the inner return map always starts
  // from a virgin SmallState, so xi never hardens the yield stress.
  const double zero4[4] = {0, 0, 0, 0};
  double ep[4];
  double xi_dummy = 0;
  const SmallResult sr = small_strain_update(p, zero4, 0.0, eps_tr, ep, &xi_dummy);

  Mat2 vv1, vv2;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) {
      vv1(i, j) = eg.v1[i] * eg.v1[j];
      vv2(i, j) = eg.v2[i] * eg.v2[j];
    }

  PlasticState next = s0;
  const double e0 = ORC_EXP(ep[0]), e1 = ORC_EXP(ep[1]);
  Mat2 m;
  for (int k = 0; k < 4; ++k) m.a[k] = e0 * vv1.a[k] + e1 * vv2.a[k];
  next.Fp = mul(m, s0.Fp);
  next.Fp_zz = ORC_EXP(ep[2]) * s0.Fp_zz;
  next.xi = s0.xi + sr.dgamma;

  const double l1n = ORC_EXP(2.0 * (eps_tr[0] - ep[0]));
  const double l2n = ORC_EXP(2.0 * (eps_tr[1] - ep[1]));
  const double a1 = sr.sigma[0] / l1n, a2 = sr.sigma[1] / l2n;
  Mat2 s_hat;
  for (int k = 0; k < 4; ++k) s_hat.a[k] = a1 * vv1.a[k] + a2 * vv2.a[k];

  const Mat2 fpn_inv = inverse(next.Fp);
  LargeResult res;
  res.P = mul(mul(mul(F, fpn_inv), s_hat), transpose(fpn_inv));
  res.dgamma = sr.dgamma;
  res.f_trial = sr.f_trial;
  res.q_trial = sr.q_trial;
  res.mises = sr.mises;
  if (s1) *s1 = next;
  return res;
}

// material.cpp:164-181: central differences, k outer / l inner, history
// frozen at s0, h = h_rel * max(1, ||F||_F).
void large_strain_tangent(const PlasticityParams& p, const PlasticState& s0, const Mat2& F,
                          double h_rel, double out[16]) {
  const double h = h_rel * std::max(1.0, frob_norm(F));
  for (int k = 0; k < 2; ++k)
    for (int l = 0; l < 2; ++l) {
      Mat2 fp = F, fm = F;
      fp(k, l) += h;
      fm(k, l) -= h;
      const Mat2 pp = large_strain_update(p, s0, fp, nullptr).P;
      const Mat2 pm = large_strain_update(p, s0, fm, nullptr).P;
      const int col = k + 2 * l;
      for (int j = 0; j < 2; ++j)
        for (int i = 0; i < 2; ++i) out[(i + 2 * j) + 4 * col] = (pp(i, j) - pm(i, j)) / (2.0 * h);
    }
}

}  // namespace orc
