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

#ifndef CPH_NB_SMALLT
#define CPH_NB_SMALLT 1   // T <= 4: the lane's LJ row in registers, FSEL-selected (A/B: 0 = shared-memory table)
#endif

#ifndef CPH_NB_R2CLAMP
#define CPH_NB_R2CLAMP 1   // packed path: out-of-range entries via r^2 = 1e30 instead of two selects (A/B switch)
#endif

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
  // Entries past a lane's own (padded) count point at the lane's own atom a box diagonal away
  // (kPadCode: r > r_c, masked), so the loads are unconditional; a whole tile (32 bytes per lane, one
  // sector) is fetched at once and the next tile is prefetched while this one computes.
  const uint32_t self = (uint32_t)(valid ? i : 0) | ((uint32_t)ti << kEntryTypeShift) |
                        (kPadCode << kEntryImgShift);
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
  const uint32_t self = (uint32_t)(valid ? i : 0) | ((uint32_t)ti << kEntryTypeShift) | (kPadCode << kEntryImgShift);
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
    const bool ina = r2.x < rc2, inb = r2.y < rc2;        // padding entries: r^2 = |L|^2 (kPadCode)
#if CPH_NB_R2CLAMP
    // an entry outside (0, r_c) gets r^2 = 1e30: e^{-b^2 r^2}, r^-6 (flushed) and hence its
    // potential and force come out exactly zero, so the two selects per entry after the
    // arithmetic are not needed (ALU pipe; same sums as masking)
    const float2 r2m = f2(ina ? r2.x : 1e30f, inb ? r2.y : 1e30f);
#else
    const float2 r2m = r2;
#endif
    const float2 rinv = f2(rsqrtf(r2m.x), rsqrtf(r2m.y));
    const float2 r2inv = __fmul2_rn(rinv, rinv);
    const float2 r6 = __fmul2_rn(__fmul2_rn(r2inv, r2inv), r2inv);
    const float2 flj = __fmul2_rn(r6, __ffma2_rn(c12, r6, c6));
    const float2 den = __ffma2_rn(pbeta2, __fmul2_rn(r2m, rinv), one2);
    const float2 t = f2(__fdividef(1.0f, den.x), __fdividef(1.0f, den.y));
    const float2 zz = __fmul2_rn(r2m, kexp2);
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
#if !CPH_NB_R2CLAMP
    qe = f2(ina ? qe.x : 0.f, inb ? qe.y : 0.f);
    fs = f2(ina ? fs.x : 0.f, inb ? fs.y : 0.f);
#endif
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
      if (CPH_NB_SMALLT && kp.T <= 4) nb_atom_x2<true, true>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
      else nb_atom_x2<true, false>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
    }
    else nb_atom<false, true>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
  } else {
    if (energy) nb_atom<true, false>(kp, d, xq, s_ljf, s_lje, s_shift, r, i, valid, xi, ti, lslot, n, nmax, &elj, &ere, &eex);
    else if (kNbPacked && kp.nb_packed) {
      if (CPH_NB_SMALLT && kp.T <= 4) nb_atom_x2<false, true>(kp, d, xq, s_c6n, s_c12, shn, r, i, valid, xi, ti, lslot, n, nmax);
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

// erf corrections of atom i's excluded pairs (any distance; R12): F_i += f q_i q_j
// (2 beta/sqrt(pi) e^{-b^2 r^2} - erf(beta r)/r) (x_i - x_j) / r^2, phi_i -= q_j erf(beta r)/r
template <bool D64>
__device__ __forceinline__ void excl_correction(const KParams &kp, const DevBufs &d, int r, float4 xi, int orig,
                                                float *fx, float *fy, float *fz, float *phx, double *phxd) {
  const float beta = kp.beta, c2b = kp.two_beta_sqrtpi, qs = kp.fcoul * xi.w;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;
  const float Lx = kp.L[0], Ly = kp.L[1], Lz = kp.L[2];
  const float iLx = kp.invL[0], iLy = kp.invL[1], iLz = kp.invL[2];
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
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
    const float erf_r = rinv - erfc_poly(t) * ez * rinv;
    const float qj = xj.w;
    *phx -= qj * erf_r;
    if (D64) *phxd -= (double)(qj * erf_r);
    const float fs = qs * qj * (c2b * ez - erf_r) * rinv * rinv;
    *fx = fmaf(fs, dx, *fx);
    *fy = fmaf(fs, dy, *fy);
    *fz = fmaf(fs, dz, *fz);
  }
}

// ---- cluster-pair kernel (cph_params.pair_list = 2) ---------------------------
// One warp per super-cluster (32 consecutive atoms of a cell column, 4 i-clusters of 8).  Lane
// l = 8 b + a holds i-atom a of every i-cluster s (slot first + 8 s + a) and, per list entry,
// j-atom b of the entry's j-cluster (slot 4 J + b, loaded once per entry: the warp reads 64
// contiguous bytes).  The entry's mask word s has bit l set iff (first + 8 s + a, 4 J + b) is a
// canonical pair (each unordered pair once, exclusions removed); i-clusters s and s+1 are
// evaluated together with the paired FP32 instructions (FFMA2 / FMUL2 / FADD2) and skipped when
// both masks are empty (warp-uniform).  Same pair arithmetic as nb_atom_x2 (r < r_c inside the
// mask).  i-side F and phi accumulate in registers for the whole list; the j-side sums of an
// entry are reduced over the 8 lanes of a j-atom with shuffles and added with one float4
// reduction per j-atom; at the end the i sums are reduced over b and each lane adds its own
// atom's (plus its exclusion corrections).  f_nb is cleared before the launch.
template <bool ENERGY>
__device__ __forceinline__ void nb_cluster_warp(const KParams &kp, const DevBufs &d, const float2 *__restrict__ s_ljf,
                                                const float2 *__restrict__ s_lje, const ShiftTab &shn, int r,
                                                size_t sidx, int first, int ni, double *e_lj, double *e_real,
                                                double *e_excl) {
  const int lane = threadIdx.x & 31, a = lane & 7;
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  const int2 *meta = d.meta + (size_t)r * kp.Nst;
  float4 *fnb = d.f_nb + (size_t)r * kp.Nst;
  float4 xi[4];
  int trow[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int l = 8 * s + a;
    xi[s] = l < ni ? xq[first + l] : make_float4(0.f, 0.f, 0.f, 0.f);
    trow[s] = l < ni ? (meta[first + l].y & 0xFF) * kp.T : 0;
  }
  const float fc = kp.fcoul;
  float2 nix[2], niy[2], niz[2], qi[2], qif[2];
#pragma unroll
  for (int P = 0; P < 2; ++P) {
    nix[P] = f2(-xi[2 * P].x, -xi[2 * P + 1].x);
    niy[P] = f2(-xi[2 * P].y, -xi[2 * P + 1].y);
    niz[P] = f2(-xi[2 * P].z, -xi[2 * P + 1].z);
    qi[P] = f2(xi[2 * P].w, xi[2 * P + 1].w);
    qif[P] = f2(fc * xi[2 * P].w, fc * xi[2 * P + 1].w);
  }
  // i sums (F, phi), packed over the i-clusters (2P, 2P+1); the displacement used is
  // d_n = x_j' - x_i, so the i force is -sum fs d_n and the j force +sum fs d_n
  float2 fx[2] = {f2(0.f, 0.f), f2(0.f, 0.f)}, fy[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
  float2 fz[2] = {f2(0.f, 0.f), f2(0.f, 0.f)}, ph[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
  double elj = 0.0, ere = 0.0;
  const float rc2 = kp.rc2;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;
  const float2 kexp2 = f2(kexp, kexp);
  const float2 pbeta2 = f2(kErfcP * kp.beta, kErfcP * kp.beta);
  const float2 c2b2 = f2(kp.two_beta_sqrtpi, kp.two_beta_sqrtpi);
  const float2 one2 = f2(1.f, 1.f);
  const int ne = min(d.cl_n[sidx], kp.clcap);
  const uint32_t *CJ = d.cl_j + sidx * kp.clcap;
  const uint4 *CM = d.cl_m + sidx * kp.clcap;
  const int b = lane >> 3;
  // two-deep software pipeline: the entry after next and the next entry's j atom are loaded
  // while the current entry computes
  uint32_t cj_n = 0u, cj_nn = 0u;
  uint4 m_n = make_uint4(0u, 0u, 0u, 0u), m_nn = m_n;
  float4 xj_n = make_float4(0.f, 0.f, 0.f, 0.f);
  int tj_n = 0;
  if (ne > 0) {
    cj_n = __ldcs(CJ);
    m_n = __ldcs(CM);
    const int j = 4 * (int)(cj_n & kClJMask) + b;
    xj_n = xq[j];
    tj_n = meta[j].y & 0xFF;
  }
  if (ne > 1) { cj_nn = __ldcs(CJ + 1); m_nn = __ldcs(CM + 1); }
  for (int e = 0; e < ne; ++e) {
    const uint32_t cj = cj_n;
    const uint4 m = m_n;
    const float4 xjr = xj_n;
    const int tj = tj_n;
    cj_n = cj_nn;
    m_n = m_nn;
    if (e + 1 < ne) {
      const int jn = 4 * (int)(cj_n & kClJMask) + b;
      xj_n = xq[jn];
      tj_n = meta[jn].y & 0xFF;
    }
    if (e + 2 < ne) { cj_nn = __ldcs(CJ + e + 2); m_nn = __ldcs(CM + e + 2); }
    const int j = 4 * (int)(cj & kClJMask) + b;
    const float4 sh = shn.s[cj >> kEntryImgShift];
    const float xjx = xjr.x + sh.x, xjy = xjr.y + sh.y, xjz = xjr.z + sh.z, qj = xjr.w;
    const float2 jx = f2(xjx, xjx), jy = f2(xjy, xjy), jz = f2(xjz, xjz), qj2 = f2(qj, qj);
    float2 gx = f2(0.f, 0.f), gy = f2(0.f, 0.f), gz = f2(0.f, 0.f), gp = f2(0.f, 0.f);
#pragma unroll
    for (int P = 0; P < 2; ++P) {
      const uint32_t m0 = P ? m.z : m.x, m1 = P ? m.w : m.y;
      if ((m0 | m1) == 0u) continue;
      const float2 dx = __fadd2_rn(jx, nix[P]), dy = __fadd2_rn(jy, niy[P]), dz = __fadd2_rn(jz, niz[P]);
      const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      const bool ina = ((m0 >> lane) & 1u) && r2.x < rc2 && r2.x > 0.f;
      const bool inb = ((m1 >> lane) & 1u) && r2.y < rc2 && r2.y > 0.f;
      const float2 rinv = f2(rsqrtf(r2.x), rsqrtf(r2.y));
      const float2 r2inv = __fmul2_rn(rinv, rinv);
      const float2 r6 = __fmul2_rn(__fmul2_rn(r2inv, r2inv), r2inv);
      const float2 la = s_ljf[trow[2 * P] + tj], lb = s_ljf[trow[2 * P + 1] + tj];   // (-6 c6, 12 c12)
      const float2 flj = __fmul2_rn(r6, __ffma2_rn(f2(la.y, lb.y), r6, f2(la.x, lb.x)));
      const float2 den = __ffma2_rn(pbeta2, __fmul2_rn(r2, rinv), one2);
      const float2 t = f2(__fdividef(1.0f, den.x), __fdividef(1.0f, den.y));
      const float2 zz = __fmul2_rn(r2, kexp2);
      const float2 ez = f2(exp2f(zz.x), exp2f(zz.y));
      float2 pa = f2(-1.348251700e-01f, -1.348251700e-01f);
      pa = __ffma2_rn(pa, t, f2(4.629509449e-01f, 4.629509449e-01f));
      pa = __ffma2_rn(pa, t, f2(-3.302423954e-01f, -3.302423954e-01f));
      pa = __ffma2_rn(pa, t, f2(3.610785306e-01f, 3.610785306e-01f));
      pa = __ffma2_rn(pa, t, f2(9.128254652e-02f, 9.128254652e-02f));
      pa = __ffma2_rn(pa, t, f2(1.782859266e-01f, 1.782859266e-01f));
      pa = __ffma2_rn(pa, t, f2(1.870171428e-01f, 1.870171428e-01f));
      pa = __ffma2_rn(pa, t, f2(1.844524294e-01f, 1.844524294e-01f));
      pa = __fmul2_rn(pa, t);                                           // erfc(beta r) exp(beta^2 r^2)
      float2 er = __fmul2_rn(__fmul2_rn(pa, ez), rinv);                 // erfc(beta r) / r
      // fs = [f q_i q_j (erfc/r + 2 beta/sqrt(pi) e^{-b^2 r^2}) + 12 c12/r^12 - 6 c6/r^6] / r^2
      float2 fs = __fmul2_rn(__ffma2_rn(__fmul2_rn(qif[P], qj2), __ffma2_rn(c2b2, ez, er), flj), r2inv);
      er = f2(ina ? er.x : 0.f, inb ? er.y : 0.f);
      fs = f2(ina ? fs.x : 0.f, inb ? fs.y : 0.f);
      ph[P] = __ffma2_rn(qj2, er, ph[P]);
      gp = __ffma2_rn(qi[P], er, gp);
      fx[P] = __ffma2_rn(fs, dx, fx[P]);
      fy[P] = __ffma2_rn(fs, dy, fy[P]);
      fz[P] = __ffma2_rn(fs, dz, fz[P]);
      gx = __ffma2_rn(fs, dx, gx);
      gy = __ffma2_rn(fs, dy, gy);
      gz = __ffma2_rn(fs, dz, gz);
      if (ENERGY) {
        const float2 ca = s_lje[trow[2 * P] + tj], cb = s_lje[trow[2 * P + 1] + tj];   // (c6, c12)
        elj += ina ? (double)(r6.x * fmaf(ca.y, r6.x, -ca.x)) : 0.0;
        elj += inb ? (double)(r6.y * fmaf(cb.y, r6.y, -cb.x)) : 0.0;
        ere += (double)qif[P].x * (double)(qj * er.x) + (double)qif[P].y * (double)(qj * er.y);
      }
    }
    // j-side: sum over the 8 lanes of j-atom b, one float4 reduction
    float vx = gx.x + gx.y, vy = gy.x + gy.y, vz = gz.x + gz.y, vp = gp.x + gp.y;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      vx += __shfl_xor_sync(0xffffffffu, vx, o);
      vy += __shfl_xor_sync(0xffffffffu, vy, o);
      vz += __shfl_xor_sync(0xffffffffu, vz, o);
      vp += __shfl_xor_sync(0xffffffffu, vp, o);
    }
    if (a == 0) atomicAdd(&fnb[j], make_float4(vx, vy, vz, vp));
  }
  // i-side: sum over b (lanes a, a+8, a+16, a+24), then lane 8 b + a takes i-cluster s = b
#pragma unroll
  for (int P = 0; P < 2; ++P)
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      fx[P].x += __shfl_xor_sync(0xffffffffu, fx[P].x, o);
      fx[P].y += __shfl_xor_sync(0xffffffffu, fx[P].y, o);
      fy[P].x += __shfl_xor_sync(0xffffffffu, fy[P].x, o);
      fy[P].y += __shfl_xor_sync(0xffffffffu, fy[P].y, o);
      fz[P].x += __shfl_xor_sync(0xffffffffu, fz[P].x, o);
      fz[P].y += __shfl_xor_sync(0xffffffffu, fz[P].y, o);
      ph[P].x += __shfl_xor_sync(0xffffffffu, ph[P].x, o);
      ph[P].y += __shfl_xor_sync(0xffffffffu, ph[P].y, o);
    }
  const bool hiP = b >> 1, odd = b & 1;
  const float2 sx = hiP ? fx[1] : fx[0], sy = hiP ? fy[1] : fy[0], sz = hiP ? fz[1] : fz[0], sp = hiP ? ph[1] : ph[0];
  float ffx = -(odd ? sx.y : sx.x), ffy = -(odd ? sy.y : sy.x), ffz = -(odd ? sz.y : sz.x);
  float fphi = odd ? sp.y : sp.x;
  if (ENERGY) {
    *e_lj = elj;
    *e_real = ere;
  }
  if (lane < ni) {
    const int i = first + lane;
    const float4 xs = xq[i];
    float phx = 0.f;
    double phxd = 0.0;
    excl_correction<ENERGY>(kp, d, r, xs, meta[i].x, &ffx, &ffy, &ffz, &phx, &phxd);
    atomicAdd(&fnb[i], make_float4(ffx, ffy, ffz, fphi + phx));
    if (ENERGY) *e_excl = 0.5 * (double)kp.fcoul * (double)xs.w * phxd;
  }
}

#ifndef CPH_CL_MINB
#define CPH_CL_MINB 4
#endif

__global__ void __launch_bounds__(128, CPH_CL_MINB) k_nb_cluster(KParams kp, DevBufs d, int step_offset, int r0,
                                                                 const ShiftTab shn) {
  extern __shared__ float2 s_lj[];
  float2 *s_ljf = s_lj;                              // (-6 c6, 12 c12)
  float2 *s_lje = s_lj + kp.T * kp.T;                // (c6, c12)
  for (int t = threadIdx.x; t < kp.T * kp.T; t += blockDim.x) {
    const float2 c = d.ljtab[t];
    s_ljf[t] = make_float2(-c.x, c.y);
    s_lje[t] = make_float2(c.x / 6.0f, c.y / 12.0f);
  }
  __syncthreads();
  const int r = r0 + blockIdx.y;
  const int id = blockIdx.x * 4 + (threadIdx.x >> 5);
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  if (id >= kp.nsc) return;
  const size_t sidx = (size_t)r * kp.nsc + id;
  const int ni = d.sc_ni[sidx];
  if (ni == 0) return;
  const int first = d.sc_first[sidx];
  double elj = 0.0, ere = 0.0, eex = 0.0;
  if (energy) nb_cluster_warp<true>(kp, d, s_ljf, s_lje, shn, r, sidx, first, ni, &elj, &ere, &eex);
  else nb_cluster_warp<false>(kp, d, s_ljf, s_lje, shn, r, sidx, first, ni, &elj, &ere, &eex);
  if (energy) {
    // warp sums (warps of a CTA may have returned early: no block-wide reduction)
    elj = warp_sum_d(elj);
    ere = warp_sum_d(ere);
    eex = warp_sum_d(eex);
    if ((threadIdx.x & 31) == 0) {
      double *e = d.erec + ((size_t)(m & 1) * kp.R + r) * kNE;
      atomicAdd(e + CPH_E_LJ, elj);
      atomicAdd(e + CPH_E_REAL, ere);
      atomicAdd(e + CPH_E_EXCL, eex);
    }
  }
}

// fp64 real-space potential of the lambda atoms in cluster mode (dV/dlambda at 2e-5; the pair
// kernel's j-side sums are fp32 reductions): one warp per lambda atom over its full canonical
// row (k_build_lam_list), same pair arithmetic as nb_atom, the per-pair values summed in fp64,
// plus the exclusion corrections.
__global__ void __launch_bounds__(128) k_phi_lam(KParams kp, DevBufs d, const ShiftTab shn) {
  const int r = blockIdx.y, k = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= kp.nlam) return;
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  const int orig = d.g_atoms[k];
  const int i = d.iperm[(size_t)r * kp.N + orig];
  const float4 xi = xq[i];
  const int n = min(d.lam_n[(size_t)r * kp.nlam + k], kp.cap);
  const uint32_t *L = d.lam_nbl + ((size_t)r * kp.nlam + k) * kp.cap;
  const float rc2 = kp.rc2;
  const float kexp = -kp.beta * kp.beta * 1.4426950408889634f;
  const float pbeta = kErfcP * kp.beta;
  double s = 0.0;
  for (int e = lane; e < n; e += 32) {
    const uint32_t ent = L[e];
    const float4 xj = xq[ent & kEntryJMask];
    const float4 sh = shn.s[ent >> kEntryImgShift];
    const float dx = (xj.x + sh.x) - xi.x, dy = (xj.y + sh.y) - xi.y, dz = (xj.z + sh.z) - xi.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    if (!(r2 < rc2 && r2 > 0.f)) continue;
    const float rinv = rsqrtf(r2);
    const float t = __fdividef(1.0f, fmaf(pbeta, r2 * rinv, 1.0f));
    const float ez = exp2f(r2 * kexp);
    s += (double)(erfc_poly(t) * (xj.w * ez) * rinv);
  }
  s = warp_sum_d(s);
  if (lane == 0) {
    float fx = 0.f, fy = 0.f, fz = 0.f, phx = 0.f;
    double phxd = 0.0;
    excl_correction<true>(kp, d, r, xi, orig, &fx, &fy, &fz, &phx, &phxd);
    d.phi64_nb[(size_t)r * kp.nlam + k] = s + phxd;
  }
}

int launch_nonbonded(Ctx &c, cudaStream_t s, int step_offset) {
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  ShiftTab shn;
  for (int code = 0; code < 27; ++code)
    shn.s[code] = make_float4(-c.kp.L[0] * (float)(code / 9 - 1), -c.kp.L[1] * (float)((code / 3) % 3 - 1),
                              -c.kp.L[2] * (float)(code % 3 - 1), 0.f);
  if (c.kp.pair_mode == 1) {
    cudaMemsetAsync(c.d.f_nb, 0, sizeof(float4) * (size_t)c.kp.R * c.kp.Nst, s);
    k_nb_cluster<<<dim3((c.kp.nsc + 3) / 4, c.kp.R), 128, 2 * sizeof(float2) * c.kp.T * c.kp.T, s>>>(
        c.kp, c.d, step_offset, 0, shn);
    if (c.kp.nlam) k_phi_lam<<<dim3((c.kp.nlam + 3) / 4, c.kp.R), 128, 0, s>>>(c.kp, c.d, shn);
    return c.kp.nlam ? 2 : 1;
  }
  k_nonbonded<<<grid, 128, 3 * sizeof(float2) * c.kp.T * c.kp.T, s>>>(c.kp, c.d, step_offset, 0, shn);
  return 1;
}

}  // namespace cph
