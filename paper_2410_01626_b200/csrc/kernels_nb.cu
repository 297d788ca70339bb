// Real-space Ewald + Lennard-Jones pair kernel that also accumulates phi_i.
//
// One thread per (sorted) atom i walks its full neighbour list, so forces and potentials are
// accumulated in registers with no atomics and in a fixed order (run-to-run deterministic).
// For r < rc:
//   E_ij  = c12/r^12 - c6/r^6 + f q_i q_j erfc(beta r)/r
//   phi_i += q_j erfc(beta r)/r
//   F_i   += [f q_i q_j (erfc(beta r)/r + 2 beta/sqrt(pi) e^{-beta^2 r^2}) + 12 c12/r^12 - 6 c6/r^6] / r^2 * (x_i - x_j)
// Excluded pairs (any distance) get the erf correction -f q_i q_j erf(beta r)/r.
// List entries carry the periodic image of j fixed at the last rebuild (positions are
// wrapped into the box then), so no per-pair minimum-image arithmetic is needed.
// Warps that contain a lambda atom also accumulate phi in fp64 (dV/dlambda at 2e-5; BASELINE
// "fp64 lambda reductions"); on energy steps the per-atom sums are fp64 as well.
// Compiled with -ftz=true: no denormal fix-ups around MUFU.RSQ / RCP / EX2.
#include "cph_device.cuh"

namespace cph {

#ifndef CPH_NB_MINB
#define CPH_NB_MINB 7   // CTAs per SM the register budget is sized for (A/B: 6 and 8 slower)
#endif

template <bool ENERGY, bool PHI64>
__device__ __forceinline__ void nb_atom(const KParams &kp, const DevBufs &d, const float4 *__restrict__ xq,
                                        const float2 *__restrict__ ljf, const float2 *__restrict__ lje,
                                        const float4 *__restrict__ shift, int r, int i, bool valid,
                                        float4 xi, int ti, int lslot, int n, int nmax,
                                        double *e_lj, double *e_real, double *e_excl) {
  const float qif = kp.fcoul * xi.w;
  float fx = 0.f, fy = 0.f, fz = 0.f, phi = 0.f;
  double phid = 0.0, elj = 0.0;        // fp64 only in lambda warps / on energy steps
  // 8-entry tiles nbl[k/8][i][k%8] (kernels_list.cu): one 16-byte load per 4 neighbours; the
  // builder pads a lane's last tile with its own slot
  const uint4 *L = reinterpret_cast<const uint4 *>(d.nbl + (size_t)r * kp.cap * kp.Nst) + 2 * (size_t)i;
  const size_t tstride = 2 * (size_t)kp.Nst;
  const float2 *ljrow = ljf + ti * kp.T;
  const float2 *ljerow = lje + ti * kp.T;
  const float rc2 = kp.rc2, beta = kp.beta, c2b = kp.two_beta_sqrtpi;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;   // exp(-b^2 r^2) = 2^(kexp r^2)
  const float pbeta = kErfcP * kp.beta;
  constexpr int U = 4;                 // neighbours in flight per lane (half a list tile)
  // Entries past a lane's own (padded) count point at the lane's own atom with zero shift
  // (r2 = 0, masked), so the loads are unconditional; a whole tile (32 bytes per lane, one
  // sector) is fetched at once and the next tile is prefetched while this one computes.
  const uint32_t self = (uint32_t)(valid ? i : 0) | ((uint32_t)ti << kEntryTypeShift) |
                        (13u << kEntryImgShift);
  const uint4 selfv = make_uint4(self, self, self, self);
  uint4 ta = selfv, tb = selfv;
  if (n > 0) { ta = __ldcs(L); tb = __ldcs(L + 1); }
  auto chunk = [&](const uint4 ev) {
    const uint32_t e[U] = {ev.x, ev.y, ev.z, ev.w};
    float4 xj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xj[u] = __ldg(&xq[(int)(e[u] & kEntryJMask)]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4 sh = shift[e[u] >> kEntryImgShift];
      const float dx = (xi.x - xj[u].x) + sh.x;
      const float dy = (xi.y - xj[u].y) + sh.y;
      const float dz = (xi.z - xj[u].z) + sh.z;
      const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const bool in = (r2 < rc2) && (r2 > 0.0f);
      const float rinv = rsqrtf(r2);
      const float r2inv = rinv * rinv;
      const float2 c = ljrow[(e[u] >> kEntryTypeShift) & kEntryTypeMask];   // (6 c6, 12 c12)
      const float r6 = r2inv * r2inv * r2inv;
      const float flj = r6 * fmaf(c.y, r6, -c.x);
      const float t = __fdividef(1.0f, fmaf(pbeta, r2 * rinv, 1.0f));   // 1/(1 + p beta r)
      const float ez = exp2f(r2 * kexp);                                 // exp(-beta^2 r^2)
      const float bq = xj[u].w * ez;                                     // q_j e^{-z^2}
      const float qe = in ? erfc_poly(t) * bq * rinv : 0.f;              // q_j erfc(beta r)/r
      const float fs = in ? fmaf(qif, fmaf(c2b, bq, qe), flj) * r2inv : 0.f;
      phi += qe;
      fx = fmaf(fs, dx, fx);
      fy = fmaf(fs, dy, fy);
      fz = fmaf(fs, dz, fz);
      if (PHI64 || ENERGY) phid += (double)qe;
      if (ENERGY) {
        const float2 ce = ljerow[(e[u] >> kEntryTypeShift) & kEntryTypeMask];   // (c6, c12)
        elj += in ? (double)(r6 * fmaf(ce.y, r6, -ce.x)) : 0.0;
      }
    }
  };
  for (int k0 = 0; k0 < nmax; k0 += 8) {
    const uint4 ca = ta, cb = tb;
    const int kn = k0 + 8;
    if (kn < n) {
      const uint4 *Lt = L + (size_t)(kn >> 3) * tstride;
      ta = __ldcs(Lt);
      tb = __ldcs(Lt + 1);
    } else {
      ta = selfv;
      tb = selfv;
    }
    chunk(ca);
    if (k0 + 4 < nmax) chunk(cb);
  }
  // exclusion corrections (solute atoms only; most atoms have none)
  float phx = 0.f;
  double phxd = 0.0;
  if (valid) {
    const float Lx = kp.L[0], Ly = kp.L[1], Lz = kp.L[2];
    const float iLx = kp.invL[0], iLy = kp.invL[1], iLz = kp.invL[2];
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
      const float ez = exp2f(r2 * kexp);
      const float erf_r = rinv - erfc_poly(t) * ez * rinv;   // erf(beta r)/r
      const float qj = xj.w;
      phx -= qj * erf_r;
      if (PHI64 || ENERGY) phxd -= (double)(qj * erf_r);
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
    *e_lj = 0.5 * elj;
    *e_real = 0.5 * (double)kp.fcoul * (double)xi.w * phid;
    *e_excl = 0.5 * (double)kp.fcoul * (double)xi.w * phxd;
  }
}

__global__ void __launch_bounds__(128, CPH_NB_MINB) k_nonbonded(KParams kp, DevBufs d, int step_offset) {
  // LJ tables sized T*T (dynamic shared memory): the rest of the SM's 256 KB stays L1 cache
  // for the neighbour-position gathers
  extern __shared__ float2 s_lj[];
  float2 *s_ljf = s_lj;                              // (6 c6, 12 c12) for forces
  float2 *s_lje = s_lj + kp.T * kp.T;                // (c6, c12) for energies
  __shared__ float4 s_shift[27];                    // image shift L * (kx, ky, kz)
  for (int t = threadIdx.x; t < kp.T * kp.T; t += blockDim.x) {
    const float2 c = d.ljtab[t];
    s_ljf[t] = c;
    s_lje[t] = make_float2(c.x / 6.0f, c.y / 12.0f);
  }
  if (threadIdx.x < 27) {
    const int code = threadIdx.x;
    s_shift[code] = make_float4(kp.L[0] * (float)(code / 9 - 1), kp.L[1] * (float)((code / 3) % 3 - 1),
                                kp.L[2] * (float)(code % 3 - 1), 0.f);
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
  const int n = valid ? min(d.nnb[idx], kp.cap) : 0;   // overflow is flagged by the builder
  const int nmax = __reduce_max_sync(0xffffffffu, n);
  const bool warp_lam = __any_sync(0xffffffffu, lslot >= 0);
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  double elj = 0.0, ere = 0.0, eex = 0.0;
  if (warp_lam) {
    if (energy) nb_atom<true, true>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else nb_atom<false, true>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
  } else {
    if (energy) nb_atom<true, false>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else nb_atom<false, false>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
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
  k_nonbonded<<<grid, 128, 2 * sizeof(float2) * c.kp.T * c.kp.T, s>>>(c.kp, c.d, step_offset);
  return 1;
}

}  // namespace cph
