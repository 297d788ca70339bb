// Host-side Partition Function Correction (R2, R6).
//
// Z_prot = int_{lp<0.5} e^{-beta V}, Z_deprot = int_{lp>=0.5} e^{-beta V} over the whole
// wall-bounded range, V = Vdw + VpH (Vmm excluded).  The lambda=1 well depth d1
// is solved so that G_deprot - G_prot = ln10 kT (pKa - pH) (bisection); His-like sites solve
// (d1_p, d1_t) for the two micro free energies (Newton).  Targets out of reach of the single
// well-depth correction saturate at +-80 kJ/mol (R22).  Composite Gauss-Legendre quadrature
// with panels split at the spline knots and wall onsets, where the integrand is analytic.
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

// Panels end at the spline knots and wall onsets (the integrand is analytic inside); the
// steep quartic-wall intervals get more sub-panels.  Beyond -0.35 / 1.35 the integrand is
// below 1e-30 of its peak.
Nodes make_nodes(int sub, int order) {
  static const double brk[] = {-0.35, -0.1, 0.0, 0.5, 1.0, 1.1, 1.35};
  static const int wsub[] = {3, 1, 2, 2, 1, 3};
  std::vector<double> gx, gw;
  gauss_legendre(order, gx, gw);
  Nodes nd;
  for (int b = 0; b + 1 < (int)(sizeof(brk) / sizeof(brk[0])); ++b) {
    const double a0 = brk[b], a1 = brk[b + 1];
    const int nsub = sub * wsub[b];
    for (int s = 0; s < nsub; ++s) {
      const double c = a0 + (a1 - a0) * s / nsub, e = a0 + (a1 - a0) * (s + 1) / nsub;
      for (int k = 0; k < order; ++k) {
        nd.x.push_back(0.5 * (e - c) * gx[k] + 0.5 * (e + c));
        nd.w.push_back(0.5 * (e - c) * gw[k]);
      }
    }
  }
  return nd;
}

double free_energy_2state(const Nodes &nd, double h, double d1, double g, double kT, double kw) {
  double zp = 0.0, zd = 0.0;
  for (size_t k = 0; k < nd.x.size(); ++k) {
    double v, dv;
    vdw_eval(nd.x[k], h, d1, kw, &v, &dv);
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

bool pfc_two_state(double h, double pKa, double pH, double T, double kw, double *d1, std::string *err) {
  static const Nodes nd = make_nodes(6, 24);
  const double kT = kBoltz * T;
  const double target = delta_g(pKa, pH, T);
  *d1 = root_or_bound([&](double x) { return free_energy_2state(nd, h, x, target, kT, kw) - target; });
  (void)err;
  return true;
}

bool pfc_three_state(double h, const double pKa3[3], double pH, double T, double kw, double *d1p,
                     double *d1t, std::string *err) {
  static const Nodes nd = make_nodes(2, 20);
  const int n = (int)nd.x.size();
  const double kT = kBoltz * T;
  const double gd = delta_g(pKa3[1], pH, T), ge = delta_g(pKa3[2], pH, T);
  // coupling kernel of VpH = lp [(1-lt) gd + lt ge]
  std::vector<double> Kpt((size_t)n * n);
  for (int p = 0; p < n; ++p)
    for (int t = 0; t < n; ++t)
      Kpt[(size_t)p * n + t] = std::exp(-nd.x[p] * ((1.0 - nd.x[t]) * gd + nd.x[t] * ge) / kT);
  std::vector<double> a(n), b(n);
  auto quad = [&](double dp, double dt, double out[2]) {
    for (int k = 0; k < n; ++k) {
      double v, dv;
      vdw_eval(nd.x[k], h, dp, kw, &v, &dv);
      a[k] = nd.w[k] * std::exp(-v / kT);
      vdw_eval(nd.x[k], h, dt, kw, &v, &dv);
      b[k] = nd.w[k] * std::exp(-v / kT);
    }
    double zp = 0.0, zdl = 0.0, zep = 0.0;
    for (int p = 0; p < n; ++p) {
      double s_lo = 0.0, s_hi = 0.0;
      const double *row = &Kpt[(size_t)p * n];
      for (int t = 0; t < n; ++t) {
        const double c = b[t] * row[t];
        if (nd.x[t] < 0.5) s_lo += c; else s_hi += c;
      }
      if (nd.x[p] < 0.5) zp += a[p] * (s_lo + s_hi);
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
