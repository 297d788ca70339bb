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
#include <algorithm>
#include <cstdlib>

#include "cph_device.cuh"

namespace cph {

#ifndef CPH_NB_PACKED
#define CPH_NB_PACKED 1   // FFMA2 pair path for non-lambda warps on non-energy steps (A/B switch)
#endif
constexpr bool kNbPacked = CPH_NB_PACKED;

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

// -shift of the 27 image codes as a kernel parameter: indexed per entry it is read through the
// constant cache (LDC), off the LSU data path that the neighbour gathers saturate
struct ShiftTab {
  float4 s[27];
};

// The hot path (no lambda atom in the warp, not an energy step) with the arithmetic of two
// list entries packed into the sm_100 paired FP32 instructions (FFMA2 / FMUL2 / FADD2: one issue
// slot for two lanes' worth of FP32 work); rsqrt / rcp / ex2 stay scalar on the MUFU pipe.  Same
// formulas and rounding as nb_atom (each packed op is the scalar op, element-wise).
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// address of the entry's neighbour: base + 16 * slot in one IMAD.WIDE.U32
__device__ __forceinline__ const float4 *slot_ptr(const char *base, uint32_t e) {
  const float4 *p;
  asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(p) : "r"(e & kEntryJMask), "l"(base));
  return p;
}

template <bool PHI64, bool SMALLT>
__device__ __forceinline__ void nb_atom_x2(const KParams &kp, const DevBufs &d, const float4 *__restrict__ xq,
                                           const float *__restrict__ c6n, const float *__restrict__ c12t,
                                           const ShiftTab &shn, int r, int i, bool valid, float4 xi, int ti,
                                           int lslot, int n, int nmax) {
  // d_n = x_j - shift - x_i = -(x_i - x_j + shift): the packed adds need no negation; the force
  // sum is negated once at the end
  const float2 nxi = f2(-xi.x, -xi.y);
  const float nzi = -xi.z;
  const float2 qif = f2(kp.fcoul * xi.w, kp.fcoul * xi.w);
  float2 fxy = f2(0.f, 0.f), phi = f2(0.f, 0.f);
  float fzs = 0.f;
  double phid = 0.0;                    // lambda warps: phi_i in fp64 (dV/dlambda at 2e-5)
  const uint4 *L = reinterpret_cast<const uint4 *>(d.nbl + (size_t)r * kp.cap * kp.Nst) + 2 * (size_t)i;
  const size_t tstride = 2 * (size_t)kp.Nst;
  const int lrow = ti * kp.T;
  // T <= 4 LJ types (the synthetic systems): the lane's LJ row lives in registers and is
  // selected with FSELs, so the pair loop issues no shared-memory load for it (the kernel is
  // bound by LSU wavefronts: global gathers + shared loads)
  float r6n[4] = {0.f, 0.f, 0.f, 0.f}, r12[4] = {0.f, 0.f, 0.f, 0.f};
  if (SMALLT) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t < kp.T) { r6n[t] = c6n[lrow + t]; r12[t] = c12t[lrow + t]; }
  }
  auto ljsel = [&](uint32_t e, float &v6, float &v12) {
    // the two type bits tested in place (one predicate-writing LOP3 each)
    const bool hi = e & (2u << kEntryTypeShift), od = e & (1u << kEntryTypeShift);
    v6 = hi ? (od ? r6n[3] : r6n[2]) : (od ? r6n[1] : r6n[0]);
    v12 = hi ? (od ? r12[3] : r12[2]) : (od ? r12[1] : r12[0]);
  };
  const float rc2 = kp.rc2;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;
  const float2 kexp2 = f2(kexp, kexp);
  const float2 pbeta2 = f2(kErfcP * kp.beta, kErfcP * kp.beta);
  const float2 c2b2 = f2(kp.two_beta_sqrtpi, kp.two_beta_sqrtpi);
  const float2 one2 = f2(1.f, 1.f);
  const uint32_t self = (uint32_t)(valid ? i : 0) | ((uint32_t)ti << kEntryTypeShift) | (13u << kEntryImgShift);
  const uint4 selfv = make_uint4(self, self, self, self);
  uint4 ta = selfv, tb = selfv;
  if (n > 0) { ta = __ldcs(L); tb = __ldcs(L + 1); }
  // the replica's base address as an opaque 64-bit value: j is then added with one
  // IMAD.WIDE.U32 instead of a 64-bit index add + LEA pair per entry
  const char *xqb;
  asm("mov.b64 %0, %1;" : "=l"(xqb) : "l"(xq));
  auto pair = [&](uint32_t ea, uint32_t eb) {
    const float4 xa = __ldg(slot_ptr(xqb, ea));
    const float4 xb = __ldg(slot_ptr(xqb, eb));
    const float4 sa = shn.s[ea >> kEntryImgShift], sb = shn.s[eb >> kEntryImgShift];
    float2 c6, c12;                                                        // (-6 c6, 12 c12)
    if (SMALLT) {
      ljsel(ea, c6.x, c12.x);
      ljsel(eb, c6.y, c12.y);
    } else {
      const int la = lrow + (int)((ea >> kEntryTypeShift) & kEntryTypeMask);
      const int lb = lrow + (int)((eb >> kEntryTypeShift) & kEntryTypeMask);
      c6 = f2(c6n[la], c6n[lb]);
      c12 = f2(c12t[la], c12t[lb]);
    }
    const float2 da = __fadd2_rn(__fadd2_rn(f2(xa.x, xa.y), f2(sa.x, sa.y)), nxi);
    const float2 db = __fadd2_rn(__fadd2_rn(f2(xb.x, xb.y), f2(sb.x, sb.y)), nxi);
    const float dza = (xa.z + sa.z) + nzi, dzb = (xb.z + sb.z) + nzi;
    const float2 qa = __fmul2_rn(da, da), qb = __fmul2_rn(db, db);
    const float2 r2 = f2(fmaf(dza, dza, qa.x + qa.y), fmaf(dzb, dzb, qb.x + qb.y));
    const bool ina = (r2.x < rc2) && (r2.x > 0.0f), inb = (r2.y < rc2) && (r2.y > 0.0f);
    const float2 rinv = f2(rsqrtf(r2.x), rsqrtf(r2.y));
    const float2 r2inv = __fmul2_rn(rinv, rinv);
    const float2 r6 = __fmul2_rn(__fmul2_rn(r2inv, r2inv), r2inv);
    const float2 flj = __fmul2_rn(r6, __ffma2_rn(c12, r6, c6));
    const float2 den = __ffma2_rn(pbeta2, __fmul2_rn(r2, rinv), one2);
    const float2 t = f2(__fdividef(1.0f, den.x), __fdividef(1.0f, den.y));
    const float2 zz = __fmul2_rn(r2, kexp2);
    const float2 ez = f2(exp2f(zz.x), exp2f(zz.y));
    const float2 bq = __fmul2_rn(f2(xa.w, xb.w), ez);
    float2 pa = f2(-1.348251700e-01f, -1.348251700e-01f);
    pa = __ffma2_rn(pa, t, f2(4.629509449e-01f, 4.629509449e-01f));
    pa = __ffma2_rn(pa, t, f2(-3.302423954e-01f, -3.302423954e-01f));
    pa = __ffma2_rn(pa, t, f2(3.610785306e-01f, 3.610785306e-01f));
    pa = __ffma2_rn(pa, t, f2(9.128254652e-02f, 9.128254652e-02f));
    pa = __ffma2_rn(pa, t, f2(1.782859266e-01f, 1.782859266e-01f));
    pa = __ffma2_rn(pa, t, f2(1.870171428e-01f, 1.870171428e-01f));
    pa = __ffma2_rn(pa, t, f2(1.844524294e-01f, 1.844524294e-01f));
    pa = __fmul2_rn(pa, t);                                       // erfc(beta r) exp(beta^2 r^2)
    float2 qe = __fmul2_rn(__fmul2_rn(pa, bq), rinv);             // q_j erfc(beta r) / r
    float2 fs = __fmul2_rn(__ffma2_rn(qif, __ffma2_rn(c2b2, bq, qe), flj), r2inv);
    qe = f2(ina ? qe.x : 0.f, inb ? qe.y : 0.f);
    fs = f2(ina ? fs.x : 0.f, inb ? fs.y : 0.f);
    phi = __fadd2_rn(phi, qe);
    if (PHI64) phid += (double)qe.x + (double)qe.y;
    fxy = __ffma2_rn(f2(fs.x, fs.x), da, fxy);
    fxy = __ffma2_rn(f2(fs.y, fs.y), db, fxy);
    fzs = fmaf(fs.x, dza, fzs);
    fzs = fmaf(fs.y, dzb, fzs);
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
    pair(ca.x, ca.y);
    pair(ca.z, ca.w);
    if (k0 + 4 < nmax) {
      pair(cb.x, cb.y);
      pair(cb.z, cb.w);
    }
  }
  float ffx = -fxy.x, ffy = -fxy.y, ffz = -fzs, fphi = phi.x + phi.y;
  // exclusion corrections (solute atoms only; most atoms have none): scalar, as nb_atom
  if (valid) {
    const float beta = kp.beta, c2b = kp.two_beta_sqrtpi, qs = kp.fcoul * xi.w;
    const float Lx = kp.L[0], Ly = kp.L[1], Lz = kp.L[2];
    const float iLx = kp.invL[0], iLy = kp.invL[1], iLz = kp.invL[2];
    const int orig = d.meta[(size_t)r * kp.Nst + i].x;
    const int eb = d.excl_ptr[orig], ee = d.excl_ptr[orig + 1];
    float phx = 0.f;
    double phxd = 0.0;
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
      const float erf_r = rinv - erfc_poly(t) * ez * rinv;
      const float qj = xj.w;
      phx -= qj * erf_r;
      if (PHI64) phxd -= (double)(qj * erf_r);
      const float fs = qs * qj * (c2b * ez - erf_r) * rinv * rinv;
      ffx = fmaf(fs, dx, ffx);
      ffy = fmaf(fs, dy, ffy);
      ffz = fmaf(fs, dz, ffz);
    }
    d.f_nb[(size_t)r * kp.Nst + i] = make_float4(ffx, ffy, ffz, fphi + phx);
    if (PHI64 && lslot >= 0) d.phi64_nb[(size_t)r * kp.nlam + lslot] = phid + phxd;
  }
}

__global__ void __launch_bounds__(128, CPH_NB_MINB) k_nonbonded(KParams kp, DevBufs d, int step_offset, int r0, const ShiftTab shn) {
  // LJ tables sized T*T (dynamic shared memory): the rest of the SM's 256 KB stays L1 cache
  // for the neighbour-position gathers
  extern __shared__ float2 s_lj[];
  float2 *s_ljf = s_lj;                              // (6 c6, 12 c12) for forces
  float2 *s_lje = s_lj + kp.T * kp.T;                // (c6, c12) for energies
  float *s_c6n = reinterpret_cast<float *>(s_lj + 2 * kp.T * kp.T);   // -6 c6 (packed path)
  float *s_c12 = s_c6n + kp.T * kp.T;                                  // 12 c12 (packed path)
  __shared__ float4 s_shift[27];                    // image shift L * (kx, ky, kz)
  for (int t = threadIdx.x; t < kp.T * kp.T; t += blockDim.x) {
    const float2 c = d.ljtab[t];
    s_ljf[t] = c;
    s_lje[t] = make_float2(c.x / 6.0f, c.y / 12.0f);
    s_c6n[t] = -c.x;
    s_c12[t] = c.y;
  }
  if (threadIdx.x < 27) {
    const int code = threadIdx.x;
    s_shift[code] = make_float4(kp.L[0] * (float)(code / 9 - 1), kp.L[1] * (float)((code / 3) % 3 - 1),
                                kp.L[2] * (float)(code % 3 - 1), 0.f);
  }
  __syncthreads();
  const int r = r0 + blockIdx.y;
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
    else if (kNbPacked && kp.nb_packed) {
      if (kp.T <= 4) nb_atom_x2<true, true>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
      else nb_atom_x2<true, false>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
    }
    else nb_atom<false, true>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
  } else {
    if (energy) nb_atom<true, false>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else if (kNbPacked && kp.nb_packed) {
      if (kp.T <= 4) nb_atom_x2<false, true>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
      else nb_atom_x2<false, false>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
    }
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
  ShiftTab shn;
  for (int code = 0; code < 27; ++code)
    shn.s[code] = make_float4(-c.kp.L[0] * (float)(code / 9 - 1), -c.kp.L[1] * (float)((code / 3) % 3 - 1),
                              -c.kp.L[2] * (float)(code % 3 - 1), 0.f);
  k_nonbonded<<<grid, 128, 3 * sizeof(float2) * c.kp.T * c.kp.T, s>>>(c.kp, c.d, step_offset, 0, shn);
  return 1;
}

}  // namespace cph
