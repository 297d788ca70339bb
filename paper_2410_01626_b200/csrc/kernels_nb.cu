// Real-space Ewald + Lennard-Jones pair kernel that also accumulates phi_i.
//
// One thread per (sorted) atom i walks its full neighbour list, so forces and potentials are
// accumulated in registers with no atomics and in a fixed order (run-to-run deterministic).
// For r < rc:
//   E_ij  = c12/r^12 - c6/r^6 + f q_i q_j erfc(beta r)/r
//   phi_i += q_j erfc(beta r)/r
//   F_i   += [f q_i q_j (erfc(beta r)/r + 2 beta/sqrt(pi) e^{-beta^2 r^2}) + 12 c12/r^12 - 6 c6/r^6] / r^2 * (x_i - x_j)
// Excluded pairs (any distance) get the erf correction -f q_i q_j erf(beta r)/r.
// Warps that contain a lambda atom accumulate phi in fp64 as well (dV/dlambda needs it at
// the 2e-5 level; BASELINE "fp64 lambda reductions").  Energies are evaluated on energy
// steps only (E_real = 1/2 f sum_i q_i phi_i, so only LJ needs a per-pair energy).
#include "cph_device.cuh"

namespace cph {

template <bool ENERGY, bool PHI64>
__device__ __forceinline__ void nb_atom(const KParams &kp, const DevBufs &d, const float4 *__restrict__ xq,
                                        const float4 *__restrict__ lj, int r, int i, bool valid,
                                        float4 xi, int ti, int lslot, int n, int nmax,
                                        double *e_lj, double *e_real, double *e_excl) {
  const float qif = kp.fcoul * xi.w;
  float fx = 0.f, fy = 0.f, fz = 0.f, phi = 0.f, elj = 0.f;
  double phid = 0.0;
  const uint32_t *L = d.nbl + (size_t)r * kp.cap * kp.Nst + i;
  const float4 *ljrow = lj + ti * kp.T;
  const float Lx = kp.L[0], Ly = kp.L[1], Lz = kp.L[2];
  const float iLx = kp.invL[0], iLy = kp.invL[1], iLz = kp.invL[2];
  const float rc2 = kp.rc2, beta = kp.beta, c2b = kp.two_beta_sqrtpi;
  const float nlog2e = -1.4426950408889634f;
#pragma unroll 2
  for (int k = 0; k < nmax; ++k) {
    if (k < n) {
      const uint32_t e = __ldcs(L + (size_t)k * kp.Nst);
      const int j = (int)(e & 0xFFFFFFu);
      const int tj = (int)(e >> 24);
      const float4 xj = __ldg(xq + j);
      float dx = xi.x - xj.x, dy = xi.y - xj.y, dz = xi.z - xj.z;
      dx -= Lx * rintf(dx * iLx);
      dy -= Ly * rintf(dy * iLy);
      dz -= Lz * rintf(dz * iLz);
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const bool in = r2 < rc2;
      const float rinv = rsqrtf(r2);
      const float r2inv = rinv * rinv;
      const float4 c = ljrow[tj];                       // (6 c6, 12 c12, c6, c12)
      const float r6 = r2inv * r2inv * r2inv;
      const float flj = r6 * fmaf(c.y, r6, -c.x);
      const float z = beta * (r2 * rinv);
      const float t = __fdividef(1.0f, fmaf(kErfcP, z, 1.0f));
      const float ez = exp2f(z * z * nlog2e);
      const float erfc_r = erfc_poly(t) * ez * rinv;
      const float qj = xj.w;
      const float qe = in ? qj * erfc_r : 0.f;
      const float fs = in ? fmaf(qif, fmaf(qj * c2b, ez, qe), flj) * r2inv : 0.f;
      phi += qe;
      fx = fmaf(fs, dx, fx);
      fy = fmaf(fs, dy, fy);
      fz = fmaf(fs, dz, fz);
      if (PHI64) phid += (double)qe;
      if (ENERGY) elj += in ? r6 * fmaf(c.w, r6, -c.z) : 0.f;
    }
  }
  // exclusion corrections (solute atoms only; most atoms have none)
  float phx = 0.f;
  double phxd = 0.0;
  if (valid) {
    const int orig = d.meta[(size_t)r * kp.Nst + i].x;
    const int eb = d.excl_ptr[orig], ee = d.excl_ptr[orig + 1];
    for (int e = eb; e < ee; ++e) {
      const int js = d.iperm[(size_t)r * kp.N + d.excl_idx[e]];
      const float4 xj = xq[js];
      float dx = xi.x - xj.x, dy = xi.y - xj.y, dz = xi.z - xj.z;
      dx -= Lx * rintf(dx * iLx);
      dy -= Ly * rintf(dy * iLy);
      dz -= Lz * rintf(dz * iLz);
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float rinv = rsqrtf(r2);
      const float z = beta * (r2 * rinv);
      const float t = __fdividef(1.0f, fmaf(kErfcP, z, 1.0f));
      const float ez = exp2f(z * z * nlog2e);
      const float erf_r = rinv - erfc_poly(t) * ez * rinv;   // erf(beta r)/r
      const float qj = xj.w;
      phx -= qj * erf_r;
      if (PHI64) phxd -= (double)(qj * erf_r);
      const float fs = qif * qj * (c2b * ez - erf_r) * rinv * rinv;
      fx = fmaf(fs, dx, fx);
      fy = fmaf(fs, dy, fy);
      fz = fmaf(fs, dz, fz);
    }
    const size_t idx = (size_t)r * kp.Nst + i;
    d.f_nb[idx] = make_float4(fx, fy, fz, phi + phx);
    if (PHI64 && lslot >= 0) d.phi64_nb[(size_t)r * kp.nlam + lslot] = phid + phxd;
  }
  if (ENERGY && valid) {
    *e_lj = 0.5 * (double)elj;
    *e_real = 0.5 * (double)qif * (double)phi;
    *e_excl = 0.5 * (double)qif * (double)phx;
  }
}

__global__ void __launch_bounds__(128) k_nonbonded(KParams kp, DevBufs d, int step_offset) {
  __shared__ float4 s_lj[kMaxTypes * kMaxTypes];
  for (int t = threadIdx.x; t < kp.T * kp.T; t += blockDim.x) {
    const float2 c = d.ljtab[t];                // (6 c6, 12 c12)
    s_lj[t] = make_float4(c.x, c.y, c.x / 6.0f, c.y / 12.0f);
  }
  __syncthreads();
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < kp.N;
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  const size_t idx = (size_t)r * kp.Nst + (valid ? i : 0);
  const float4 xi = d.xyzq[idx];
  const int2 mi = d.meta[idx];
  const int ti = mi.y & 0xFF;
  const int lslot = valid ? (mi.y >> 8) - 1 : -1;
  const int n = valid ? d.nnb[idx] : 0;
  const int nmax = __reduce_max_sync(0xffffffffu, n);
  const bool warp_lam = __any_sync(0xffffffffu, lslot >= 0);
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  double elj = 0.0, ere = 0.0, eex = 0.0;
  if (warp_lam) {
    if (energy) nb_atom<true, true>(kp, d, xq, s_lj, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else nb_atom<false, true>(kp, d, xq, s_lj, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
  } else {
    if (energy) nb_atom<true, false>(kp, d, xq, s_lj, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else nb_atom<false, false>(kp, d, xq, s_lj, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
  }
  if (energy) {
    double *e = d.erec + ((size_t)(m & 1) * kp.R + r) * kNE;
    block_atomic_add_d(elj, e + CPH_E_LJ);
    block_atomic_add_d(ere, e + CPH_E_REAL);
    block_atomic_add_d(eex, e + CPH_E_EXCL);
  }
}

int launch_nonbonded(Ctx &c, cudaStream_t s, int step_offset) {
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_nonbonded<<<grid, 128, 0, s>>>(c.kp, c.d, step_offset);
  return 1;
}

}  // namespace cph
