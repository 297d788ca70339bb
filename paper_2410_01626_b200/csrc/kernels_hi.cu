// Hamiltonian interpolation (Eq. 1 literally; SURVEY §8(f) f4;
// DESIGN.md R31).
//
// E_HI = E_CI + sum_g C_g with, per lambda-group g (forms s = A..D, weights w_s of Eq. 2),
//   C = 1/2 sum_s w_s M_ss - 1/2 w^T M w,   M_uv = q^u^T G q^v over the group's atoms,
// G the Ewald Coulomb kernel: real space (erfc inside r_c for non-excluded pairs, -erf for
// excluded ones), self (-2 beta/sqrt(pi)) and the exact reciprocal sum over the half space
// 2 g(m) cos(2 pi m.r), g(m) = exp(-pi^2 m^2/beta^2)/(pi V m^2).  Forces: with
// c = 1/2 diag(w) - 1/2 w w^T and T_u = sum_v c_uv S_v(m),
//   F_k^rec = 4 pi f sum_m 2g(m) m Im(e^{i theta_k} sum_u q_k^u conj(T_u)).
// k_hi_recip: one CTA per (m-slice, group, replica); per-atom e^{2 pi i k x/L} tables in
// shared memory (fp64 sincos, stored fp32), structure factors and M in fp64, partial sums
// added atomically.  k_hi_finish: one warp per (group, replica): real-space / self part,
// C and dC/dlambda, forces added to f_nb; clears the accumulators for the next step.
#include <algorithm>

#include "cph_device.cuh"

namespace cph {

constexpr int kHiMaxAtoms = 32;

// Forces are accumulated in registers for the atom window [a0, a0 + NF) (groups of more than
// 16 atoms take two passes); the structure factors always cover all ng atoms; M is summed in
// the first pass only.
template <int NF>
__device__ void hi_recip_body(const KParams &kp, const DevBufs &d, int r, int g, int k0, int ng, const float *q4,
                              const float2 *tab, const int *koff, const int *kstride, const float c[16], int a0,
                              bool do_M) {
  double M[10];
#pragma unroll
  for (int u = 0; u < 10; ++u) M[u] = 0.0;
  float F[NF][3];
#pragma unroll
  for (int a = 0; a < NF; ++a) F[a][0] = F[a][1] = F[a][2] = 0.f;
  const int nf = min(NF, ng - a0);
  const float ilx = kp.invL[0], ily = kp.invL[1], ilz = kp.invL[2];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kp.hi_nm; i += gridDim.x * blockDim.x) {
    const int4 mk = d.hi_m[i];
    const float w = d.hi_w[i];
    double Sr[4] = {0, 0, 0, 0}, Si[4] = {0, 0, 0, 0};
    for (int a = 0; a < ng; ++a) {
      const float2 ex = tab[koff[0] + a * kstride[0] + mk.x];
      const float2 ey = tab[koff[1] + a * kstride[1] + mk.y];
      const float2 ez = tab[koff[2] + a * kstride[2] + mk.z];
      const float xr = ex.x * ey.x - ex.y * ey.y, xi = ex.x * ey.y + ex.y * ey.x;
      const float er = xr * ez.x - xi * ez.y, ei = xr * ez.y + xi * ez.x;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Sr[u] = fma((double)q4[a * 4 + u], (double)er, Sr[u]);
        Si[u] = fma((double)q4[a * 4 + u], (double)ei, Si[u]);
      }
    }
    if (do_M) {
      int t = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = u; v < 4; ++v, ++t) M[t] = fma((double)w, Sr[u] * Sr[v] + Si[u] * Si[v], M[t]);
    }
    float Tr[4], Ti[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int v = 0; v < 4; ++v) { ar += c[u * 4 + v] * Sr[v]; ai += c[u * 4 + v] * Si[v]; }
      Tr[u] = (float)ar;
      Ti[u] = (float)ai;
    }
    const float mx = mk.x * ilx, my = mk.y * ily, mz = mk.z * ilz;
#pragma unroll
    for (int b = 0; b < NF; ++b) {
      if (b >= nf) break;
      const int a = a0 + b;
      const float2 ex = tab[koff[0] + a * kstride[0] + mk.x];
      const float2 ey = tab[koff[1] + a * kstride[1] + mk.y];
      const float2 ez = tab[koff[2] + a * kstride[2] + mk.z];
      const float xr = ex.x * ey.x - ex.y * ey.y, xi = ex.x * ey.y + ex.y * ey.x;
      const float er = xr * ez.x - xi * ez.y, ei = xr * ez.y + xi * ez.x;
      // z = sum_u q_a^u conj(T_u); Im(e z)
      float zr = 0.f, zi = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) { zr = fmaf(q4[a * 4 + u], Tr[u], zr); zi = fmaf(-q4[a * 4 + u], Ti[u], zi); }
      const float im = w * (er * zi + ei * zr);
      F[b][0] = fmaf(im, mx, F[b][0]);
      F[b][1] = fmaf(im, my, F[b][1]);
      F[b][2] = fmaf(im, mz, F[b][2]);
    }
  }
  // block reduction: M (fp64) and forces (fp32), then global atomics
  __shared__ double sM[10];
  __shared__ float sF[NF * 3];
  if (threadIdx.x < 10) sM[threadIdx.x] = 0.0;
  for (int t = threadIdx.x; t < NF * 3; t += blockDim.x) sF[t] = 0.f;
  __syncthreads();
  if (do_M) {
#pragma unroll
    for (int u = 0; u < 10; ++u) {
      const double v = warp_sum_d(M[u]);
      if ((threadIdx.x & 31) == 0) atomicAdd(&sM[u], v);
    }
  }
#pragma unroll
  for (int b = 0; b < NF; ++b) {
    if (b >= nf) break;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const float v = warp_sum_f(F[b][x]);
      if ((threadIdx.x & 31) == 0) atomicAdd(&sF[b * 3 + x], v);
    }
  }
  __syncthreads();
  if (do_M && threadIdx.x < 10) atomicAdd(&d.hi_M[((size_t)r * kp.G + g) * 10 + threadIdx.x], sM[threadIdx.x]);
  for (int t = threadIdx.x; t < nf * 3; t += blockDim.x)
    atomicAdd(&d.hi_F[((size_t)r * kp.nlam + k0 + a0) * 3 + t], sF[t]);
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_hi_recip(KParams kp, DevBufs d) {
  const int g = blockIdx.y, r = blockIdx.z;
  const int k0 = d.g_ptr[g], ng = d.g_ptr[g + 1] - k0;
  __shared__ float q4[kHiMaxAtoms * 4];
  __shared__ float c[16];
  __shared__ int koff[3], kstride[3];
  extern __shared__ float2 tab[];
  const int c0 = d.g_cptr[g];
  const size_t ic = (size_t)r * kp.C + c0;
  const double lp = d.lam[ic], lt = d.g_kind[g] == 3 ? d.lam[ic + 1] : 0.0;
  if (threadIdx.x < 16) {
    const double w[4] = {(1 - lp) * (1 - lt), (1 - lp) * lt, lp * (1 - lt), lp * lt};
    const int u = threadIdx.x >> 2, v = threadIdx.x & 3;
    c[threadIdx.x] = (float)((u == v ? 0.5 * w[u] : 0.0) - 0.5 * w[u] * w[v]);
  }
  if (threadIdx.x < 3) {
    const int s = 2 * kp.hi_kmax[threadIdx.x] + 1;
    kstride[threadIdx.x] = s;
    // table of dimension x: [ng][2 kmax + 1], offset so that index kmax + k -> tab[.. + k]
    int off = 0;
    for (int e = 0; e < (int)threadIdx.x; ++e) off += ng * (2 * kp.hi_kmax[e] + 1);
    koff[threadIdx.x] = off + kp.hi_kmax[threadIdx.x];
  }
  for (int t = threadIdx.x; t < ng * 4; t += blockDim.x) q4[t] = (float)d.g_q[(size_t)k0 * 4 + t];
  __syncthreads();
  // e^{2 pi i k x / L}, k in [-kmax, kmax], fp64 phase reduction
  for (int dim = 0; dim < 3; ++dim) {
    const int km = kp.hi_kmax[dim], s = 2 * km + 1;
    for (int t = threadIdx.x; t < ng * s; t += blockDim.x) {
      const int a = t / s, k = t % s - km;
      const int slot = d.iperm[(size_t)r * kp.N + d.g_atoms[k0 + a]];
      const float4 x = d.xyzq[(size_t)r * kp.Nst + slot];
      const double xd = dim == 0 ? x.x : (dim == 1 ? x.y : x.z);
      double ph = (double)k * xd / kp.Ld[dim];
      ph -= rint(ph);
      double sn, cs;
      sincospi(2.0 * ph, &sn, &cs);
      tab[koff[dim] - km + a * s + (k + km)] = make_float2((float)cs, (float)sn);
    }
  }
  __syncthreads();
  float cl[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) cl[t] = c[t];
  if (ng <= 8) hi_recip_body<8>(kp, d, r, g, k0, ng, q4, tab, koff, kstride, cl, 0, true);
  else {
    hi_recip_body<16>(kp, d, r, g, k0, ng, q4, tab, koff, kstride, cl, 0, true);
    if (ng > 16) hi_recip_body<16>(kp, d, r, g, k0, ng, q4, tab, koff, kstride, cl, 16, false);
  }
}

__global__ void __launch_bounds__(32) k_hi_finish(KParams kp, DevBufs d, int step_offset) {
  const int g = blockIdx.x, r = blockIdx.y, lane = threadIdx.x;
  const int k0 = d.g_ptr[g], ng = d.g_ptr[g + 1] - k0;
  const int kind = d.g_kind[g], c0 = d.g_cptr[g];
  const size_t ic = (size_t)r * kp.C + c0;
  const double lp = d.lam[ic], lt = kind == 3 ? d.lam[ic + 1] : 0.0;
  const double w[4] = {(1 - lp) * (1 - lt), (1 - lp) * lt, lp * (1 - lt), lp * lt};
  const double dwp[4] = {-(1 - lt), -lt, 1 - lt, lt};
  const double dwt[4] = {-(1 - lp), 1 - lp, -lp, lp};
  double cm[16];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) cm[u * 4 + v] = (u == v ? 0.5 * w[u] : 0.0) - 0.5 * w[u] * w[v];
  __shared__ float4 sx[kHiMaxAtoms];
  __shared__ double sq[kHiMaxAtoms * 4];
  __shared__ float sF[kHiMaxAtoms * 3];
  __shared__ int sslot[kHiMaxAtoms];
  if (lane < ng) {
    const int slot = d.iperm[(size_t)r * kp.N + d.g_atoms[k0 + lane]];
    sslot[lane] = slot;
    sx[lane] = d.xyzq[(size_t)r * kp.Nst + slot];
#pragma unroll
    for (int u = 0; u < 4; ++u) sq[lane * 4 + u] = d.g_q[(size_t)(k0 + lane) * 4 + u];
  }
  for (int t = lane; t < kHiMaxAtoms * 3; t += 32) sF[t] = 0.f;
  __syncwarp();
  const double beta = kp.beta_d, rc2 = (double)kp.rc2;
  const double c2b = 2.0 * beta / 1.7724538509055160273;
  double M[10];
#pragma unroll
  for (int u = 0; u < 10; ++u) M[u] = 0.0;
  for (int p = lane; p < ng * ng; p += 32) {
    const int i = p / ng, j = p % ng;
    double G, dG = 0.0, dx = 0.0, dy = 0.0, dz = 0.0, rr = 1.0;
    if (i == j) {
      G = -c2b;
    } else {
      dx = (double)sx[i].x - sx[j].x; dy = (double)sx[i].y - sx[j].y; dz = (double)sx[i].z - sx[j].z;
      dx -= kp.Ld[0] * rint(dx / kp.Ld[0]);
      dy -= kp.Ld[1] * rint(dy / kp.Ld[1]);
      dz -= kp.Ld[2] * rint(dz / kp.Ld[2]);
      const double r2 = dx * dx + dy * dy + dz * dz;
      rr = sqrt(r2);
      const bool ex = (d.hi_excl[k0 + i] >> j) & 1u;
      const double gau = c2b * exp(-beta * beta * r2) / rr;
      if (ex) { G = -erf(beta * rr) / rr; dG = erf(beta * rr) / r2 - gau; }
      else if (r2 < rc2) { G = erfc(beta * rr) / rr; dG = -erfc(beta * rr) / r2 - gau; }
      else G = 0.0;
    }
    int t = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = u; v < 4; ++v, ++t)
        M[t] += G * (u == v ? sq[i * 4 + u] * sq[j * 4 + u] : sq[i * 4 + u] * sq[j * 4 + v] + sq[i * 4 + v] * sq[j * 4 + u]) *
                (u == v ? 1.0 : 0.5);
    if (i != j && dG != 0.0) {
      double a = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a += cm[u * 4 + v] * sq[i * 4 + u] * sq[j * 4 + v];
      const double s = -2.0 * kFCoul * a * dG / rr;
      atomicAdd(&sF[i * 3 + 0], (float)(s * dx));
      atomicAdd(&sF[i * 3 + 1], (float)(s * dy));
      atomicAdd(&sF[i * 3 + 2], (float)(s * dz));
    }
  }
#pragma unroll
  for (int u = 0; u < 10; ++u) M[u] = warp_sum_d(M[u]);
  __syncwarp();
  double *hm = d.hi_M + ((size_t)r * kp.G + g) * 10;
  if (lane == 0) {
    // full symmetric M (with f): real/self part + reciprocal part
    double Mf[16];
    int t = 0;
    for (int u = 0; u < 4; ++u)
      for (int v = u; v < 4; ++v, ++t) Mf[u * 4 + v] = Mf[v * 4 + u] = kFCoul * (M[t] + hm[t]);
    double C = 0.0, Cp = 0.0, Ct = 0.0;
    for (int u = 0; u < 4; ++u) {
      double mw = 0.0;
      for (int v = 0; v < 4; ++v) mw += Mf[u * 4 + v] * w[v];
      C += 0.5 * w[u] * Mf[u * 5] - 0.5 * w[u] * mw;
      Cp += 0.5 * dwp[u] * Mf[u * 5] - dwp[u] * mw;
      Ct += 0.5 * dwt[u] * Mf[u * 5] - dwt[u] * mw;
    }
    d.hi_dvdl[ic] = Cp;
    if (kind == 3) d.hi_dvdl[ic + 1] = Ct;
    const long long m = *d.step + step_offset;
    if (is_energy_step(m, *d.end_step, kp.nstenergy))
      atomicAdd(&d.erec[((size_t)(m & 1) * kp.R + r) * kNE + CPH_E_HI], C);
    for (int u = 0; u < 10; ++u) hm[u] = 0.0;
  }
  __syncwarp();
  if (lane < ng) {
    float *hf = d.hi_F + ((size_t)r * kp.nlam + k0 + lane) * 3;
    const float s = (float)(4.0 * kPi * kFCoul);
    float4 *f = d.f_nb + (size_t)r * kp.Nst + sslot[lane];
    atomicAdd(&f->x, sF[lane * 3 + 0] + s * hf[0]);
    atomicAdd(&f->y, sF[lane * 3 + 1] + s * hf[1]);
    atomicAdd(&f->z, sF[lane * 3 + 2] + s * hf[2]);
    hf[0] = hf[1] = hf[2] = 0.f;
  }
}

int launch_hi_recip(Ctx &c, cudaStream_t s) {
  const KParams &kp = c.kp;
  if (!kp.hi || !kp.G) return 0;
  int maxng = 0;
  for (int g = 0; g < kp.G; ++g) maxng = std::max(maxng, c.h_group_ptr[g + 1] - c.h_group_ptr[g]);
  size_t smem = 0;
  for (int e = 0; e < 3; ++e) smem += (size_t)maxng * (2 * kp.hi_kmax[e] + 1) * sizeof(float2);
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_hi_recip, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_hi_recip<<<dim3(kp.hi_nsplit, kp.G, kp.R), 256, smem, s>>>(kp, c.d);
  return 1;
}

int launch_hi_finish(Ctx &c, cudaStream_t s, int step_offset) {
  if (!c.kp.hi || !c.kp.G) return 0;
  k_hi_finish<<<dim3(c.kp.G, c.kp.R), 32, 0, s>>>(c.kp, c.d, step_offset);
  return 1;
}

}  // namespace cph
