// Real-space Ewald + Lennard-Jones pair kernel that also accumulates phi_i.
//
// One CTA per block of cells (region.cuh): the block's region (every cell within +-2 cells)
// is staged in shared memory, then each thread takes one i atom of the block and walks its
// full neighbour list, reading neighbours from shared memory (list entries are region-local
// indices).  Forces and potentials are accumulated in registers with no atomics and in a
// fixed order (run-to-run deterministic).  For r < rc:
//   E_ij  = c12/r^12 - c6/r^6 + f q_i q_j erfc(beta r)/r
//   phi_i += q_j erfc(beta r)/r
//   F_i   += [f q_i q_j (erfc(beta r)/r + 2 beta/sqrt(pi) e^{-beta^2 r^2}) + 12 c12/r^12 - 6 c6/r^6] / r^2 * (x_i - x_j)
// Excluded pairs (any distance) get the erf correction -f q_i q_j erf(beta r)/r.
// List entries carry the periodic image of j fixed at the last rebuild (positions are
// wrapped into the box then), so no per-pair minimum-image arithmetic is needed.
// Warps that contain a lambda atom also accumulate phi in fp64 (dV/dlambda at 2e-5; BASELINE
// "fp64 lambda reductions"); on energy steps the per-atom sums are fp64 as well.
// Compiled with -ftz=true: no denormal fix-ups around MUFU.RSQ / RCP / EX2.
#include "region.cuh"

namespace cph {

template <bool ENERGY, bool PHI64>
__device__ __forceinline__ void nb_atom(const KParams &kp, const DevBufs &d, const float4 *__restrict__ xs,
                                        const float4 *__restrict__ xg, const float2 *__restrict__ ljf,
                                        const float2 *__restrict__ lje, const float4 *__restrict__ shift, int r,
                                        int i, bool valid, uint32_t self_local, float4 xi, int ti, int lslot, int n,
                                        int nmax, double *e_lj, double *e_real, double *e_excl) {
  const float qif = kp.fcoul * xi.w;
  float fx = 0.f, fy = 0.f, fz = 0.f, phi = 0.f;
  double phid = 0.0, elj = 0.0;        // fp64 only in lambda warps / on energy steps
  const uint32_t *L = d.nbl + (size_t)r * kp.cap * kp.Nst + i;
  const float2 *ljrow = ljf + ti * kp.T;
  const float2 *ljerow = lje + ti * kp.T;
  const float rc2 = kp.rc2, beta = kp.beta, c2b = kp.two_beta_sqrtpi;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;   // exp(-b^2 r^2) = 2^(kexp r^2)
  const float pbeta = kErfcP * kp.beta;
  constexpr int U = 4;                 // neighbours in flight per lane
  // Entries past a lane's own count point at the lane's own atom with zero shift (r2 = 0,
  // masked), so a chunk's U loads are unconditional and the next chunk's entries are
  // prefetched while the current chunk computes.
  const uint32_t self = self_local | ((uint32_t)ti << kEntryTypeShift) | (13u << kEntryImgShift);
  uint32_t en[U];
  const int stride = kp.Nst;
#pragma unroll
  for (int u = 0; u < U; ++u) en[u] = u < n ? __ldcs(L + u * stride) : self;
  const uint32_t *Lk = L + U * stride;
  for (int k0 = 0; k0 < nmax; k0 += U, Lk += U * stride) {
    uint32_t e[U];
    float4 xj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      e[u] = en[u];
      xj[u] = xs[e[u] & kEntryJMask];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) en[u] = k0 + U + u < n ? __ldcs(Lk + u * stride) : self;
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
      const float4 xj = xg[js];
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
    *e_lj += 0.5 * elj;
    *e_real += 0.5 * (double)kp.fcoul * (double)xi.w * phid;
    *e_excl += 0.5 * (double)kp.fcoul * (double)xi.w * phxd;
  }
}

// dynamic shared memory layout of the pair kernel
__host__ __device__ inline size_t nb_smem_bytes(const KParams &kp) {
  return sizeof(float4) * (size_t)kp.rcap + 2 * sizeof(float2) * kp.T * kp.T + sizeof(float4) * 27 +
         sizeof(int) * (2 * (size_t)kp.rcells + 1 + 2 * kMaxBlockCells + 1);
}

__global__ void __launch_bounds__(512) k_nonbonded(KParams kp, DevBufs d, int step_offset) {
  extern __shared__ float4 s_x[];                                   // [rcap]
  float2 *s_ljf = reinterpret_cast<float2 *>(s_x + kp.rcap);        // (6 c6, 12 c12)
  float2 *s_lje = s_ljf + kp.T * kp.T;                              // (c6, c12)
  float4 *s_shift = reinterpret_cast<float4 *>(s_lje + kp.T * kp.T);  // L * (kx, ky, kz)
  int *s_coff = reinterpret_cast<int *>(s_shift + 27);
  int *s_cglob = s_coff + kp.rcells + 1;
  int *s_ioff = s_cglob + kp.rcells;
  int *s_iglob = s_ioff + kMaxBlockCells + 1;
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
  const int r = blockIdx.y;
  const float4 *xg = d.xyzq + (size_t)r * kp.Nst;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const Region g = block_region(kp, blockIdx.x);
  region_tables(kp, g, start, s_coff, s_cglob, s_ioff, s_iglob);
  region_stage(xg, start, g, s_coff, s_cglob, s_x, kp.rcap);
  __syncthreads();
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  const int nI = s_ioff[g.nbcells];
  const int lane = threadIdx.x & 31;
  double elj = 0.0, ere = 0.0, eex = 0.0;
  for (int t0 = threadIdx.x - lane; t0 < nI; t0 += blockDim.x) {
    const int t = t0 + lane;
    const bool valid = t < nI;
    int bc = 0, i = 0;
    uint32_t self_local = 0;
    if (valid) {
      i = block_atom_slot(s_ioff, s_iglob, start, g.nbcells, t, &bc);
      const int cz = g.b0[2] + bc % g.bw[2];
      const int cy = g.b0[1] + (bc / g.bw[2]) % g.bw[1];
      const int cx = g.b0[0] + bc / (g.bw[2] * g.bw[1]);
      self_local = (uint32_t)(s_coff[region_local(kp, g, cx, cy, cz)] + (t - s_ioff[bc]));
    }
    const size_t idx = (size_t)r * kp.Nst + i;
    const float4 xi = xg[i];
    const int2 mi = d.meta[idx];
    const int ti = mi.y & 0xFF;
    const int lslot = valid ? (mi.y >> 8) - 1 : -1;
    const int n = valid ? d.nnb[idx] : 0;
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    const bool warp_lam = __any_sync(0xffffffffu, lslot >= 0);
    if (warp_lam) {
      if (energy) nb_atom<true, true>(kp, d, s_x, xg, s_ljf, s_lje, s_shift, r, i, valid, self_local, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
      else nb_atom<false, true>(kp, d, s_x, xg, s_ljf, s_lje, s_shift, r, i, valid, self_local, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    } else {
      if (energy) nb_atom<true, false>(kp, d, s_x, xg, s_ljf, s_lje, s_shift, r, i, valid, self_local, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
      else nb_atom<false, false>(kp, d, s_x, xg, s_ljf, s_lje, s_shift, r, i, valid, self_local, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    }
  }
  if (energy) {
    double *e = d.erec + ((size_t)(m & 1) * kp.R + r) * kNE;
    block_atomic_add_d(elj, e + CPH_E_LJ);
    block_atomic_add_d(ere, e + CPH_E_REAL);
    block_atomic_add_d(eex, e + CPH_E_EXCL);
  }
}

size_t nonbonded_smem(const KParams &kp) { return nb_smem_bytes(kp); }

int launch_nonbonded(Ctx &c, cudaStream_t s, int step_offset) {
  const size_t smem = nb_smem_bytes(c.kp);
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_nonbonded, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  dim3 grid(c.kp.nblk, c.kp.R);
  k_nonbonded<<<grid, c.kp.bthreads, smem, s>>>(c.kp, c.d, step_offset);
  return 1;
}

}  // namespace cph
