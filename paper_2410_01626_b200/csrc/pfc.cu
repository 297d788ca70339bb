// Host-side Partition Function Correction (R2, R6).
//
// Recomputed after every DBO adjustment with the shifted knots.
// Z_prot = int_{lp<0.5} e^{-beta V}, Z_deprot = int_{lp>=0.5} e^{-beta V} over the whole
// wall-bounded range, V = Vdw + VpH (Vmm excluded).  The lambda=1 well depth d1
// is solved so that G_deprot - G_prot = ln10 kT (pKa - pH) (bisection); His-like sites solve
// (d1_p, d1_t) for the two micro free energies (Newton).  Targets out of reach of the single
// well-depth correction saturate at +-80 kJ/mol (R22).  Composite Gauss-Legendre quadrature
// with panels split at the spline knots and wall onsets, where the integrand is analytic.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "cph_device.cuh"

namespace cph {

namespace {

void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int k = 1; k <= n; ++k) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
      }
      const double dp = n * (z * p0 - p1) / (z * z - 1.0);
      const double dz = p0 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) {
        double q0 = 1.0, q1 = 0.0;
        for (int k = 1; k <= n; ++k) {
          const double q2 = q1;
          q1 = q0;
          q0 = ((2.0 * k - 1.0) * z * q1 - (k - 1.0) * q2) / k;
        }
        const double dq = n * (z * q0 - q1) / (z * z - 1.0);
        x[i] = z;
        w[i] = 2.0 / ((1.0 - z * z) * dq * dq);
        break;
      }
    }
  }
}

struct Nodes {
  std::vector<double> x, w;
};

// Panels end at the spline knots (the DBO well centres a0, a1 and the barrier position
// (a0+a1)/2 of the coordinate), the smoothstep ends 0 and 1 of a protonation-keyed
// tautomer barrier, the half-space split 0.5 and the wall onsets -0.1 / 1.1: the integrand
// is analytic inside each.  Interior intervals get ~4*sub panels per unit length (at least
// sub), the steep quartic-wall intervals 3*sub.  Beyond -0.35 / 1.35 the integrand is below
// 1e-30 of its peak.
Nodes make_nodes(int sub, int order, double a0, double a1) {
  std::vector<double> brk = {-0.35, -0.1, 0.0, 0.5, 1.0, 1.1, 1.35, a0, a1, 0.5 * (a0 + a1)};
  std::sort(brk.begin(), brk.end());
  std::vector<double> b;
  for (double v : brk)
    if (b.empty() || v - b.back() > 1e-12) b.push_back(v);
  std::vector<double> gx, gw;
  gauss_legendre(order, gx, gw);
  Nodes nd;
  for (size_t k = 0; k + 1 < b.size(); ++k) {
    const double lo = b[k], hi = b[k + 1];
    const bool wall = hi <= -0.1 + 1e-12 || lo >= 1.1 - 1e-12;
    const int nsub = wall ? 3 * sub : std::max(sub, (int)std::ceil((hi - lo) * 4.0 * sub - 1e-9));
    for (int s = 0; s < nsub; ++s) {
      const double c = lo + (hi - lo) * s / nsub, e = lo + (hi - lo) * (s + 1) / nsub;
      for (int q = 0; q < order; ++q) {
        nd.x.push_back(0.5 * (e - c) * gx[q] + 0.5 * (e + c));
        nd.w.push_back(0.5 * (e - c) * gw[q]);
      }
    }
  }
  return nd;
}

double free_energy_2state(const Nodes &nd, const double dw[4], double d1, double g, double kT, double kw) {
  double zp = 0.0, zd = 0.0;
  for (size_t k = 0; k < nd.x.size(); ++k) {
    double v, dv;
    vdw_eval(nd.x[k], dw[0], dw[1], dw[2], d1, kw, &v, &dv, nullptr);
    const double b = nd.w[k] * std::exp(-(v + nd.x[k] * g) / kT);
    if (nd.x[k] < 0.5) zp += b; else zd += b;
  }
  return -kT * std::log(zd / zp);
}

}  // namespace

double delta_g(double pKa, double pH, double T) { return kLn10 * kBoltz * T * (pKa - pH); }

// DESIGN.md R22: root of an increasing function on [-80, 80] kJ/mol, or the bound nearer
// to it when the target is out of reach of the single well-depth correction
constexpr double kD1Bound = 80.0;
template <class F>
double root_or_bound(F f) {
  double lo = -kD1Bound, hi = kD1Bound;
  if (f(lo) > 0.0) return lo;
  if (f(hi) < 0.0) return hi;
  for (int it = 0; it < 200 && hi - lo > 1e-13; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (f(mid) < 0.0) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

bool pfc_two_state(const double dw[4], double pKa, double pH, double T, double kw, double *d1, std::string *err) {
  const Nodes nd = make_nodes(6, 24, dw[0], dw[1]);
  const double kT = kBoltz * T;
  const double target = delta_g(pKa, pH, T);
  *d1 = root_or_bound([&](double x) { return free_energy_2state(nd, dw, x, target, kT, kw) - target; });
  (void)err;
  return true;
}

// V_t(lt; h, d1) = h U(lt) + d1 W(lt) + walls(lt) (linear in h and d1): the protonation-keyed
// tautomer barrier h(lp) enters through exp(-h(lp) U(lt) / kT), tabulated once per solve.
bool pfc_three_state(const double dwp[4], const double dwt[4], const double pKa3[3], double pH, double T,
                     double kw, double *d1p, double *d1t, std::string *err) {
  const Nodes np_ = make_nodes(2, 20, dwp[0], dwp[1]);
  const Nodes nt = make_nodes(2, 20, dwt[0], dwt[1]);
  const int n = (int)np_.x.size(), m = (int)nt.x.size();
  const double kT = kBoltz * T;
  const double gd = delta_g(pKa3[1], pH, T), ge = delta_g(pKa3[2], pH, T);
  std::vector<double> U(m), Wd(m), Wall(m);
  for (int t = 0; t < m; ++t) {
    double v0, v1, v2, dv;
    vdw_eval(nt.x[t], dwt[0], dwt[1], 0.0, 0.0, kw, &v0, &dv, nullptr);
    vdw_eval(nt.x[t], dwt[0], dwt[1], 1.0, 0.0, kw, &v1, &dv, nullptr);
    vdw_eval(nt.x[t], dwt[0], dwt[1], 0.0, 1.0, kw, &v2, &dv, nullptr);
    Wall[t] = v0;
    U[t] = v1 - v0;
    Wd[t] = v2 - v0;
  }
  // M[p][t] = exp(-(h(lp) U(lt) + VpH(lp, lt)) / kT), VpH = lp [(1-lt) gd + lt ge]
  std::vector<double> M((size_t)n * m);
  for (int p = 0; p < n; ++p) {
    double h, dh;
    tautomer_barrier(np_.x[p], dwt[2], dwt[3], &h, &dh);
    for (int t = 0; t < m; ++t)
      M[(size_t)p * m + t] = std::exp(-(h * U[t] + np_.x[p] * ((1.0 - nt.x[t]) * gd + nt.x[t] * ge)) / kT);
  }
  std::vector<double> a(n), b(m);
  auto quad = [&](double dp, double dt, double out[2]) {
    for (int k = 0; k < n; ++k) {
      double v, dv;
      vdw_eval(np_.x[k], dwp[0], dwp[1], dwp[2], dp, kw, &v, &dv, nullptr);
      a[k] = np_.w[k] * std::exp(-v / kT);
    }
    for (int t = 0; t < m; ++t) b[t] = nt.w[t] * std::exp(-(dt * Wd[t] + Wall[t]) / kT);
    double zp = 0.0, zdl = 0.0, zep = 0.0;
    for (int p = 0; p < n; ++p) {
      double s_lo = 0.0, s_hi = 0.0;
      const double *row = &M[(size_t)p * m];
      for (int t = 0; t < m; ++t) {
        const double c = b[t] * row[t];
        if (nt.x[t] < 0.5) s_lo += c; else s_hi += c;
      }
      if (np_.x[p] < 0.5) zp += a[p] * (s_lo + s_hi);
      else { zdl += a[p] * s_lo; zep += a[p] * s_hi; }
    }
    out[0] = -kT * std::log(zdl / zp) - gd;
    out[1] = -kT * std::log(zep / zp) - ge;
  };
  double x0 = 0.0, x1 = 0.0;
  for (int it = 0; it < 60; ++it) {
    double f[2], fa[2], fb[2];
    quad(x0, x1, f);
    if (std::fabs(f[0]) < 1e-12 && std::fabs(f[1]) < 1e-12) break;
    const double e = 1e-6;
    quad(x0 + e, x1, fa);
    quad(x0, x1 + e, fb);
    const double j00 = (fa[0] - f[0]) / e, j10 = (fa[1] - f[1]) / e;
    const double j01 = (fb[0] - f[0]) / e, j11 = (fb[1] - f[1]) / e;
    const double det = j00 * j11 - j01 * j10;
    if (!(std::fabs(det) > 1e-300)) break;      // unreachable / degenerate: fall back below
    double s0 = (j11 * f[0] - j01 * f[1]) / det;
    double s1 = (-j10 * f[0] + j00 * f[1]) / det;
    const double mx = std::fmax(std::fabs(s0), std::fabs(s1));
    if (mx > 10.0) { s0 *= 10.0 / mx; s1 *= 10.0 / mx; }
    x0 -= s0;
    x1 -= s1;
  }
  double f[2];
  quad(x0, x1, f);
  if (std::fabs(f[0]) < 1e-9 && std::fabs(f[1]) < 1e-9 && std::fabs(x0) <= kD1Bound && std::fabs(x1) <= kD1Bound) {
    *d1p = x0;
    *d1t = x1;
    return true;
  }
  // R22: unreachable targets -> nested saturating bisection: the tautomer split
  // G_eps - G_delta = dG_eps - dG_delta for d1_t inside, the macro deprotonation free
  // energy -kT ln(e^{-b dG_delta} + e^{-b dG_eps}) for d1_p outside
  const double macro = -kT * std::log(std::exp(-gd / kT) + std::exp(-ge / kT));
  auto inner = [&](double dp) {
    return root_or_bound([&](double dt) {
      double q[2];
      quad(dp, dt, q);
      return (q[1] + ge) - (q[0] + gd) - (ge - gd);
    });
  };
  auto outer = [&](double dp) {
    double q[2];
    quad(dp, inner(dp), q);
    const double a = q[0] + gd, b = q[1] + ge;
    return -kT * std::log(std::exp(-a / kT) + std::exp(-b / kT)) - macro;
  };
  *d1p = root_or_bound(outer);
  *d1t = inner(*d1p);
  (void)err;
  return true;
}

}  // namespace cph
