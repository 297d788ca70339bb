// Device helpers shared by the library's kernels (not by the oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "cph_internal.cuh"

namespace cph {

// ---------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11).  key = (seed lo, seed hi); counters per
// DESIGN.md R17: atoms (step, atom, 0, 0), lambda (step, coord, 1, 0).
// ---------------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ inline U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    U4 n;
    n.x = hi1 ^ c.y ^ k0; n.y = lo1; n.z = hi0 ^ c.w ^ k1; n.w = lo0;
    c = n;
  }
  return c;
}

// three fp32 standard normals for an atom (Box-Muller on u = (x + 0.5) 2^-32)
__device__ inline float3 atom_normals(uint64_t seed, uint32_t step, uint32_t atom) {
  U4 o = philox4x32_10(U4{step, atom, 0u, 0u}, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float s = 2.3283064365386963e-10f;  // 2^-32
  float u0 = ((float)o.x + 0.5f) * s, u1 = ((float)o.y + 0.5f) * s;
  float u2 = ((float)o.z + 0.5f) * s, u3 = ((float)o.w + 0.5f) * s;
  // u0 may round to 1.0f in fp32: log(1) = 0 gives a zero radius, harmless
  float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  return make_float3(r0 * c0, r0 * s0, r1 * c1);
}

// one fp64 standard normal for a lambda coordinate
__device__ inline double lambda_normal(uint64_t seed, uint32_t step, uint32_t coord) {
  U4 o = philox4x32_10(U4{step, coord, 1u, 0u}, (uint32_t)seed, (uint32_t)(seed >> 32));
  double u0 = ((double)o.x + 0.5) * 2.3283064365386963e-10;
  double u1 = ((double)o.y + 0.5) * 2.3283064365386963e-10;
  return sqrt(-2.0 * log(u0)) * cospi(2.0 * u1);
}

// ---------------------------------------------------------------------------------
// Bussi-Donadio-Parrinello velocity rescaling factor for one thermostat group
// (R27/R28): R1 and the chi^2(Nf-1) sum S come from Philox counters
// (step, k, stream, 0); S by explicit squares for Nf-1 <= 32, else 2 Gamma((Nf-1)/2)
// by Marsaglia-Tsang.  K' = K + (1-c)(Kbar (R1^2+S)/Nf - K) + 2 R1 sqrt(K Kbar/Nf (1-c) c),
// alpha = sgn(R1 + sqrt(c Nf K/((1-c) Kbar))) sqrt(K'/K), c = exp(-dt/tau).
// ---------------------------------------------------------------------------------
__device__ inline void philox_uniforms(uint64_t seed, uint32_t step, uint32_t k, uint32_t stream, double u[4]) {
  const U4 o = philox4x32_10(U4{step, k, stream, 0u}, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double s = 2.3283064365386963e-10;
  u[0] = ((double)o.x + 0.5) * s; u[1] = ((double)o.y + 0.5) * s;
  u[2] = ((double)o.z + 0.5) * s; u[3] = ((double)o.w + 0.5) * s;
}

__device__ inline double bussi_alpha(uint64_t seed, uint32_t step, uint32_t stream, double K, int nf, double kT,
                                     double c) {
  if (nf <= 0 || !(K > 0.0)) return 1.0;
  double u[4];
  philox_uniforms(seed, step, 0u, stream, u);
  const double R1 = sqrt(-2.0 * log(u[0])) * cospi(2.0 * u[1]);
  const int m = nf - 1;
  double S = 0.0;
  if (m > 0 && m <= 32) {
    for (int k = 1, left = m; left > 0; ++k) {
      philox_uniforms(seed, step, (uint32_t)k, stream, u);
      const double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
      const double z[4] = {r0 * cospi(2.0 * u[1]), r0 * sinpi(2.0 * u[1]), r1 * cospi(2.0 * u[3]),
                           r1 * sinpi(2.0 * u[3])};
      for (int q = 0; q < 4 && left > 0; ++q, --left) S += z[q] * z[q];
    }
  } else if (m > 32) {
    const double d = 0.5 * m - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * d);
    for (uint32_t k = 1;; ++k) {
      philox_uniforms(seed, step, k, stream, u);
      const double x = sqrt(-2.0 * log(u[0])) * cospi(2.0 * u[1]);
      const double t = 1.0 + cc * x;
      const double v = t * t * t;
      if (v > 0.0 && log(u[2]) < 0.5 * x * x + d - d * v + d * log(v)) { S = 2.0 * d * v; break; }
    }
  }
  const double kbar = 0.5 * nf * kT;
  const double kn = K + (1.0 - c) * (kbar * (R1 * R1 + S) / nf - K) + 2.0 * R1 * sqrt(K * kbar / nf * (1.0 - c) * c);
  double alpha = sqrt(fmax(kn, 0.0) / K);
  if (c < 1.0 && R1 + sqrt(c * nf * K / ((1.0 - c) * kbar)) < 0.0) alpha = -alpha;
  return alpha;
}

// ---------------------------------------------------------------------------------
// erfc(z) = t P(t) exp(-z^2), t = 1/(1 + p z): least-squares-minimax fit of
// erfcx(z)/t on z in [0, 4] (rel. error 3e-8 in exact arithmetic, 4e-7 in fp32).
// exp(-z^2) is shared with the Ewald force term.
// ---------------------------------------------------------------------------------
constexpr float kErfcP = 0.3275911f;
__device__ __forceinline__ float erfc_poly(float t) {
  float a = -1.348251700e-01f;
  a = fmaf(a, t, 4.629509449e-01f);
  a = fmaf(a, t, -3.302423954e-01f);
  a = fmaf(a, t, 3.610785306e-01f);
  a = fmaf(a, t, 9.128254652e-02f);
  a = fmaf(a, t, 1.782859266e-01f);
  a = fmaf(a, t, 1.870171428e-01f);
  a = fmaf(a, t, 1.844524294e-01f);
  return a * t;   // erfc(z) * exp(z^2)
}

// minimum image with the canonical fp32 formula (round-to-nearest, no contraction)
__device__ __forceinline__ float min_image_rn(float dx, float L, float invL) {
  return __fsub_rn(dx, __fmul_rn(L, rintf(__fmul_rn(dx, invL))));
}

// ---------------------------------------------------------------------------------
// Bias potential pieces (host + device, fp64).  DESIGN.md R4/R5:
//   Vdw: cubic Hermite through (0,0,0), (0.5,h,0), (1,d1,0), mirrored outside
//   [0,1], quartic walls k_w (l+0.1)^4 below -0.1 and k_w (l-1.1)^4 above 1.1.
// ---------------------------------------------------------------------------------
// Double well with DBO-movable well centres a0, a1:
// cubic Hermite knots (a0, 0), (m, h), (a1, d1), m = (a0 + a1)/2, zero slopes; mirrored about
// a0 / a1 outside [a0, a1]; quartic walls k_w (lam + 0.1)^4 below -0.1 and k_w (lam - 1.1)^4
// above 1.1 (R5, R23).  Returns V, dV/dlam and dV/dh (V is linear in h).
__host__ __device__ inline void vdw_eval(double lam, double a0, double a1, double h, double d1, double kw,
                                         double *v, double *dv, double *dh) {
  const double m = 0.5 * (a0 + a1);
  double x = lam, sgn = 1.0;
  if (lam < a0) { x = 2.0 * a0 - lam; sgn = -1.0; }
  else if (lam > a1) { x = 2.0 * a1 - lam; sgn = -1.0; }
  x = x < a0 ? a0 : (x > a1 ? a1 : x);
  double a, b, t, w;
  bool left = x <= m;
  if (left) { a = 0.0; b = h; w = m - a0; t = (x - a0) / w; }
  else { a = h; b = d1; w = a1 - m; t = (x - m) / w; }
  const double s = t * t * (3.0 - 2.0 * t);
  double val = a + (b - a) * s;
  double der = sgn * (b - a) * 6.0 * t * (1.0 - t) / w;
  if (lam < -0.1) { double q = lam + 0.1; val += kw * q * q * q * q; der += 4.0 * kw * q * q * q; }
  else if (lam > 1.1) { double q = lam - 1.1; val += kw * q * q * q * q; der += 4.0 * kw * q * q * q; }
  *v = val;
  *dv = der;
  if (dh) *dh = left ? s : 1.0 - s;
}

// barrier of a tautomer coordinate keyed by protonation, smooth in lambda_p (R25)
__host__ __device__ inline void tautomer_barrier(double lp, double hp, double hd, double *h, double *dh) {
  const double x = lp < 0.0 ? 0.0 : (lp > 1.0 ? 1.0 : lp);
  *h = hp + (hd - hp) * x * x * (3.0 - 2.0 * x);
  *dh = (lp > 0.0 && lp < 1.0) ? (hd - hp) * 6.0 * x * (1.0 - x) : 0.0;
}

__host__ __device__ inline void vmm_eval(const double *c, double lp, double lt, double *v, double *dp,
                                         double *dt) {
  double pp[6], pt[6];
  pp[0] = pt[0] = 1.0;
  for (int k = 1; k < 6; ++k) { pp[k] = pp[k - 1] * lp; pt[k] = pt[k - 1] * lt; }
  double V = 0, DP = 0, DT = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      double cab = c[a * 6 + b];
      V += cab * pp[a] * pt[b];
      if (a) DP += a * cab * pp[a - 1] * pt[b];
      if (b) DT += b * cab * pp[a] * pt[b - 1];
    }
  *v = V; *dp = DP; *dt = DT;
}

// Bias of one lambda-group (Eq. 3) at (lp, lt): returns V and
// dV/dlp, dV/dlt.  vmm36 == nullptr leaves Vmm out (the pH-independent term, e.g. for the
// replica-exchange energies).  dG = (dG_macro, dG_delta, dG_eps) at the pH; d1 = PFC depths
// of the group's coordinates; dw = DBO rows (a0, a1, h_prot, h_deprot) of its coordinates.
__host__ __device__ inline double group_bias_eval(int kind, const double *vmm36, const double *dG, const double *d1,
                                                  const double *dw, double kw, double lp, double lt, double *dp,
                                                  double *dt) {
  double vm = 0.0, vmp = 0.0, vmt = 0.0;
  if (vmm36) vmm_eval(vmm36, lp, lt, &vm, &vmp, &vmt);
  double vph, vphp, vpht;
  if (kind == 2) { vph = lp * dG[0]; vphp = dG[0]; vpht = 0.0; }
  else {
    vph = lp * ((1.0 - lt) * dG[1] + lt * dG[2]);
    vphp = (1.0 - lt) * dG[1] + lt * dG[2];
    vpht = lp * (dG[2] - dG[1]);
  }
  double vd, vdp;
  vdw_eval(lp, dw[0], dw[1], dw[2], d1[0], kw, &vd, &vdp, nullptr);
  double V = vm + vph + vd;
  *dt = 0.0;
  if (kind == 3) {
    const double *wt = dw + 4;
    double ht, dht, vd2, vdt, vdh;
    tautomer_barrier(lp, wt[2], wt[3], &ht, &dht);
    vdw_eval(lt, wt[0], wt[1], ht, d1[1], kw, &vd2, &vdt, &vdh);
    *dt = vmt + vpht + vdt;
    vdp += vdh * dht;
    V += vd2;
  }
  *dp = vmp + vphp + vdp;
  return V;
}

__device__ inline double warp_sum_d(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline float warp_sum_f(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-reduce a double into one atomicAdd (blockDim multiple of 32, <= 1024)
__device__ inline void block_atomic_add_d(double v, double *dst) {
  __shared__ double red[32];
  v = warp_sum_d(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    double s = lane < nw ? red[lane] : 0.0;
    s = warp_sum_d(s);
    if (lane == 0 && s != 0.0) atomicAdd(dst, s);
  }
  __syncthreads();
}

__device__ __forceinline__ bool is_energy_step(long long m, long long end, int nstenergy) {
  return (m % nstenergy) == 0 || m == end;
}

// ---- smooth PME B-splines (R16) -------------------------------------------------
// Grid convention: atom with scaled fractional coordinate u = K (x/L - floor(x/L)) puts weight
// M4(u - k) on grid points k = floor(u) - j, j = 0..3 (mod K); w = u - floor(u).
__device__ __forceinline__ void bspline4(const float x, const float invL, const int K, int &k0,
                                         float th[4], float dth[4]) {
  const float t = x * invL;
  const float s = t - floorf(t);
  const float u = s * (float)K;
  float fl = floorf(u);
  const float w = u - fl;
  int k = (int)fl;
  if (k >= K) k -= K;
  k0 = k;
  const float w2 = w * w, w3 = w2 * w, om = 1.0f - w;
  const float s6 = 1.0f / 6.0f;
  th[0] = w3 * s6;
  th[1] = (-3.0f * w3 + 3.0f * w2 + 3.0f * w + 1.0f) * s6;
  th[2] = (3.0f * w3 - 6.0f * w2 + 4.0f) * s6;
  th[3] = om * om * om * s6;
  dth[0] = 0.5f * w2;
  dth[1] = 0.5f * (-3.0f * w2 + 2.0f * w + 1.0f);
  dth[2] = 0.5f * (3.0f * w2 - 4.0f * w);
  dth[3] = -0.5f * om * om;
}

// fp64 phi_rec of one atom from the back-transformed grid g of its replica: the B-spline
// weighted sum over the 4x4x4 points (z rows in fp32, products with theta_x theta_y in fp64),
// spread over 16 lanes (one (x, y) row of 4 z points each, aligned 16-lane
// groups) and reduced with a fixed shuffle tree; every lane of the group returns the total.
// All 32 lanes of the warp must call it (inactive groups pass act = false).
__device__ __forceinline__ double pme_phi64_x16(const KParams &kp, const float *g, const float4 p, bool act) {
  const int ab = threadIdx.x & 15, a = ab >> 2, b = ab & 3;
  double v = 0.0;
  if (act) {
    int kx, ky, kz;
    float tx[4], ty[4], tz[4], dd[4];
    bspline4(p.x, kp.invL[0], kp.K[0], kx, tx, dd);
    bspline4(p.y, kp.invL[1], kp.K[1], ky, ty, dd);
    bspline4(p.z, kp.invL[2], kp.K[2], kz, tz, dd);
    const int ix = (kx - a + kp.K[0]) % kp.K[0];
    const int iy = (ky - b + kp.K[1]) % kp.K[1];
    const float *row = g + ((size_t)ix * kp.K[1] + iy) * kp.K[2];
    float sa = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) sa = fmaf(tz[c], __ldg(row + (kz - c + kp.K[2]) % kp.K[2]), sa);
    float txa = tx[0], tyb = ty[0];
#pragma unroll
    for (int q = 1; q < 4; ++q) { txa = a == q ? tx[q] : txa; tyb = b == q ? ty[q] : tyb; }
    v = (double)(txa * tyb) * (double)sa;
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace cph
