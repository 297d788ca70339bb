// Atom and lambda-particle integration and the lambda-group reduction.
//
// BAOAB (R9): B v += dt/2 F/m ; A x += dt/2 v ; O v = c1 v + sqrt((1-c1^2) kT/m) xi ;
// A x += dt/2 v ; forces at (x, lambda) ; B v += dt/2 F/m.  The closing B of step n is fused
// into the opening of step n+1 (FLAG_PENDING_CLOSE) and finished by k_close at the end of a
// cph_step call, so atom data is read and written once per step.
#include "cph_device.cuh"

namespace cph {

__global__ void __launch_bounds__(128) k_integrate(KParams kp, DevBufs d) {
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = *d.step;
  const long long end = *d.end_step;
  const int pending = d.flags[FLAG_PENDING_CLOSE];
  if (blockIdx.x == 0 && threadIdx.x < kNE)   // record of step n+1 starts empty
    d.erec[((size_t)((n + 1) & 1) * kp.R + r) * kNE + threadIdx.x] = 0.0;
  double ke = 0.0, kmid = 0.0;
  if (i < kp.N) {
    const size_t idx = (size_t)r * kp.Nst + i;
    float4 v = d.vel[idx];
    const float invm = v.w;
    const int2 mt = d.meta[idx];
    const int lslot = (mt.y >> 8) - 1;   // lambda atom: charge of this step from qlam (lambda_set_charges)
    const float qnew = lslot >= 0 ? (float)d.qlam[(size_t)r * kp.nlam + lslot] : 0.f;
    if (invm > 0.0f) {
      float4 x = d.xyzq[idx];
      if (lslot >= 0) x.w = qnew;
      const float4 fa = d.f_nb[idx], fb = d.f_rec[idx];
      const float fx = fa.x + fb.x, fy = fa.y + fb.y, fz = fa.z + fb.z;
      const float hk = 0.5f * kp.dt * invm;
      if (pending) {
        v.x = fmaf(hk, fx, v.x); v.y = fmaf(hk, fy, v.y); v.z = fmaf(hk, fz, v.z);
        ke = 0.5 * ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z) / invm;
      }
      v.x = fmaf(hk, fx, v.x); v.y = fmaf(hk, fy, v.y); v.z = fmaf(hk, fz, v.z);      // B
      const float hdt = 0.5f * kp.dt;
      x.x = fmaf(hdt, v.x, x.x); x.y = fmaf(hdt, v.y, x.y); x.z = fmaf(hdt, v.z, x.z);  // A
      if (kp.bussi) {
        // Bussi: the group's mid-step kinetic energy is reduced here; k_thermo rescales
        // and applies the second A (R27)
        kmid = 0.5 * ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z) / invm;
        d.xyzq[idx] = x;
        d.vel[idx] = v;
        goto done;
      }
      const int orig = mt.x;
      const float3 xi = atom_normals(d.seed[r], (uint32_t)n, (uint32_t)orig);
      const float sd = sqrtf(kp.c2_atom_kT * invm);
      v.x = fmaf(kp.c1_atom, v.x, sd * xi.x);                                           // O
      v.y = fmaf(kp.c1_atom, v.y, sd * xi.y);
      v.z = fmaf(kp.c1_atom, v.z, sd * xi.z);
      x.x = fmaf(hdt, v.x, x.x); x.y = fmaf(hdt, v.y, x.y); x.z = fmaf(hdt, v.z, x.z);  // A
      d.xyzq[idx] = x;
      d.vel[idx] = v;
    } else if (lslot >= 0) {
      d.xyzq[idx].w = qnew;
    }
  }
done:
  if (pending && is_energy_step(n, end, kp.nstenergy))
    block_atomic_add_d(ke, &d.erec[((size_t)(n & 1) * kp.R + r) * kNE + CPH_E_KE_ATOMS]);
  if (kp.bussi) {
    if (blockIdx.x == 0 && threadIdx.x == 0) d.bussi_k[((n + 1) & 1) * kp.R + r] = 0.0;   // next step's sum
    block_atomic_add_d(kmid, &d.bussi_k[(n & 1) * kp.R + r]);
  }
}

// Bussi step for the atoms of every replica: alpha from the reduced mid-step kinetic energy
// (computed once per CTA), v *= alpha, then the second A
__global__ void __launch_bounds__(128) k_thermo(KParams kp, DevBufs d) {
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = *d.step;
  __shared__ double s_alpha;
  if (threadIdx.x == 0)
    s_alpha = bussi_alpha(d.seed[r], (uint32_t)n, 2u, d.bussi_k[(n & 1) * kp.R + r], (int)kp.nf_atom, kp.kT,
                          kp.cb_atom);
  __syncthreads();
  if (i >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + i;
  float4 v = d.vel[idx];
  if (v.w > 0.0f) {
    const float a = (float)s_alpha;
    v.x *= a; v.y *= a; v.z *= a;
    float4 x = d.xyzq[idx];
    const float hdt = 0.5f * kp.dt;
    x.x = fmaf(hdt, v.x, x.x); x.y = fmaf(hdt, v.y, x.y); x.z = fmaf(hdt, v.z, x.z);  // A
    d.xyzq[idx] = x;
    d.vel[idx] = v;
  }
}

// closing half kick (kick = 1) and/or kinetic energy of the current velocities
__global__ void __launch_bounds__(128) k_close(KParams kp, DevBufs d, int kick) {
  const int r = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = *d.step;
  double ke = 0.0;
  if (i < kp.N) {
    const size_t idx = (size_t)r * kp.Nst + i;
    const int lslot = (d.meta[idx].y >> 8) - 1;   // end of a cph_step call: qlam -> xyzq.w
    if (lslot >= 0) d.xyzq[idx].w = (float)d.qlam[(size_t)r * kp.nlam + lslot];
    float4 v = d.vel[idx];
    if (v.w > 0.0f) {
      if (kick) {
        const float4 fa = d.f_nb[idx], fb = d.f_rec[idx];
        const float hk = 0.5f * kp.dt * v.w;
        v.x = fmaf(hk, fa.x + fb.x, v.x); v.y = fmaf(hk, fa.y + fb.y, v.y); v.z = fmaf(hk, fa.z + fb.z, v.z);
        d.vel[idx] = v;
      }
      ke = 0.5 * ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z) / v.w;
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) d.flags[FLAG_PENDING_CLOSE] = 0;
  block_atomic_add_d(ke, &d.erec[((size_t)(n & 1) * kp.R + r) * kNE + CPH_E_KE_ATOMS]);
}

// ---- lambda helpers ---------------------------------------------------------------------
// charges of every lambda atom of replica r from its group's (lp, lt) (Eq. 2).
// Inside a step (to_xyzq = false) only qlam is written: the all-atom force gather may still be
// reading xyzq.w of this step on the PME stream, and the next k_integrate (or k_close at the
// end of a cph_step call) copies qlam into xyzq.w.
__device__ void lambda_set_charges(const KParams &kp, const DevBufs &d, int r, bool to_xyzq = true) {
  for (int k = threadIdx.x; k < kp.nlam; k += blockDim.x) {       // one thread per lambda atom
    const int g = d.k_group[k];
    const int c0 = d.g_cptr[g];
    const double lp = d.lam[(size_t)r * kp.C + c0];
    const double lt = d.g_kind[g] == 3 ? d.lam[(size_t)r * kp.C + c0 + 1] : 0.0;
    const double wA = (1.0 - lp) * (1.0 - lt), wB = (1.0 - lp) * lt, wC = lp * (1.0 - lt), wD = lp * lt;
    const double *qs = d.g_q + 4 * (size_t)k;
    const double q = wA * qs[0] + wB * qs[1] + wC * qs[2] + wD * qs[3];
    d.qlam[(size_t)r * kp.nlam + k] = q;
    if (!to_xyzq) continue;
    const int slot = d.iperm[(size_t)r * kp.N + d.g_atoms[k]];
    d.xyzq[(size_t)r * kp.Nst + slot].w = (float)q;
  }
}

__device__ double block_sum_d(double v);

// BAOA for lambda coordinates of replica r with noise index `step`, then new charges
// (O = Langevin, or the Bussi rescaling of the replica's lambda group, R27)
__device__ void lambda_open(const KParams &kp, const DevBufs &d, int r, long long step, bool to_xyzq = true) {
  const double h = kp.dtd;
  double ke = 0.0;
  for (int c = threadIdx.x; c < kp.C; c += blockDim.x) {
    const size_t ix = (size_t)r * kp.C + c;
    const double F = -(d.dvdl_coul[ix] + d.dvdl_bias[ix]);
    double v = d.lamv[ix], l = d.lam[ix];
    v += 0.5 * h * F / kp.m_lam;                                              // B
    l += 0.5 * h * v;                                                         // A
    if (kp.bussi) {
      ke += 0.5 * kp.m_lam * v * v;
    } else {
      v = kp.c1_lam * v + kp.sd_lam * lambda_normal(d.seed[r], (uint32_t)step, (uint32_t)c);  // O
      l += 0.5 * h * v;                                                       // A
    }
    d.lamv[ix] = v;
    d.lam[ix] = l;
  }
  if (kp.bussi) {
    const double K = block_sum_d(ke);
    const double alpha = bussi_alpha(d.seed[r], (uint32_t)step, 3u, K, kp.C, kp.kT, kp.cb_lam);
    for (int c = threadIdx.x; c < kp.C; c += blockDim.x) {
      const size_t ix = (size_t)r * kp.C + c;
      const double v = alpha * d.lamv[ix];                                    // O (Bussi)
      d.lamv[ix] = v;
      d.lam[ix] += 0.5 * h * v;                                               // A
    }
  }
  __syncthreads();
  lambda_set_charges(kp, d, r, to_xyzq);
}

__device__ double block_sum_d(double v) {
  __shared__ double red[32];
  __shared__ double tot;
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double s = lane < nw ? red[lane] : 0.0;
    s = warp_sum_d(s);
    if (lane == 0) tot = s;
  }
  __syncthreads();
  const double out = tot;
  __syncthreads();
  return out;
}

// One CTA per replica.  mode 0: evaluation at create/set_state (step index = *step, no
// integration); mode 1: end of a step (index m = *step + 1): dV/dlambda, bias, closing B,
// frames, energies, then (unless m is the call's last step) the next BAOA + charges.
__global__ void __launch_bounds__(256) k_lambda_reduce(KParams kp, DevBufs d, int mode) {
  const int r = blockIdx.x;
  const long long n = *d.step;
  const long long m = mode == 1 ? n + 1 : n;
  const long long end = *d.end_step;
  const bool energy = is_energy_step(m, end, kp.nstenergy);
  const bool dyn = kp.mode == 0;
  const double f = kFCoul;
  const double V = kp.Ld[0] * kp.Ld[1] * kp.Ld[2];
  const double sqrtpi = 1.7724538509055160273;

  // per lambda atom (one thread each): potential (real + excl + recip + self) and its
  // products with dq/dlp, dq/dlt, staged in shared memory for the per-group sums.  The
  // net-charge term -pi Q/(V beta^2) is the same for every atom and every group's charge is
  // constant in lambda (sum_i dq_i/dlambda = 0, checked at create), so it adds nothing to
  // dV/dlambda; it enters the energies and cph_get_forces' phi only.
  extern __shared__ double s_dq[];            // [3 * nlam]: 2 products per atom, then phi_rec
  double *s_prec = s_dq + 2 * kp.nlam;
  // phi_rec of the lambda atoms from the back-transformed PME grid, 16 lanes per atom (the
  // all-atom force gather runs beside this kernel on the PME stream)
  for (int w0 = 0; w0 < 16 * kp.nlam; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x, k = w >> 4;
    const bool act = k < kp.nlam;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) p = d.xyzq[(size_t)r * kp.Nst + d.iperm[(size_t)r * kp.N + d.g_atoms[k]]];
    const double v = pme_phi64_x16(kp, d.grid + (size_t)r * kp.K3, p, act);
    if (act && (w & 15) == 0) s_prec[k] = v;
  }
  __syncthreads();
  double qs = 0.0, qq = 0.0;                  // total lambda charge and sum of squares
  for (int k = threadIdx.x; k < kp.nlam; k += blockDim.x) {
    const size_t ix = (size_t)r * kp.nlam + k;
    const double q = d.qlam[ix];
    qs += q;
    qq += q * q;
    const double prec = s_prec[k];
    const double phi = d.phi64_nb[ix] + prec - 2.0 * kp.beta_d / sqrtpi * q;
    d.phi_lam[ix] = phi;
    const int g = d.k_group[k];
    const size_t ic = (size_t)r * kp.C + d.g_cptr[g];
    const double lp = d.lam[ic];
    const double lt = d.g_kind[g] == 3 ? d.lam[ic + 1] : 0.0;
    const double *q4 = d.g_q + 4 * (size_t)k;
    s_dq[2 * k] = ((1.0 - lt) * (q4[2] - q4[0]) + lt * (q4[3] - q4[1])) * phi;
    s_dq[2 * k + 1] = ((1.0 - lp) * (q4[1] - q4[0]) + lp * (q4[3] - q4[2])) * phi;
  }
  __syncthreads();
  // per group: Coulomb dV/dlambda (fixed-order sum over the group's atoms) and bias
  double ebias = 0.0;
  for (int g = threadIdx.x; g < kp.G; g += blockDim.x) {
    const int kind = d.g_kind[g];
    const int c0 = d.g_cptr[g];
    const size_t ic = (size_t)r * kp.C + c0;
    const double lp = d.lam[ic];
    const double lt = kind == 3 ? d.lam[ic + 1] : 0.0;
    double sp = 0.0, st = 0.0;
    for (int k = d.g_ptr[g]; k < d.g_ptr[g + 1]; ++k) {
      sp += s_dq[2 * k];
      st += s_dq[2 * k + 1];
    }
    // bias (Eq. 3): Vmm + VpH + Vdw, double wells with the DBO parameters of each coordinate
    double bp, bt;
    ebias += group_bias_eval(kind, d.vmm + 36 * (size_t)g, d.g_dG + ((size_t)r * kp.G + g) * 3, d.d1 + ic,
                             d.dw + ic * 4, kp.wall_k, lp, lt, &bp, &bt);
    // Hamiltonian interpolation: + dC/dlambda of the group (kernels_hi.cu)
    d.dvdl_coul[ic] = f * sp + (kp.hi ? d.hi_dvdl[ic] : 0.0);
    d.dvdl_bias[ic] = bp;
    if (kind == 3) {
      d.dvdl_coul[ic + 1] = f * st + (kp.hi ? d.hi_dvdl[ic + 1] : 0.0);
      d.dvdl_bias[ic + 1] = bt;
    }
  }
  // dV/dlambda visible to the block; the reductions only on energy steps
  double Q = 0.0, Q2 = 0.0;
  if (energy) {
    ebias = block_sum_d(ebias);
    Q = kp.Q_fixed + block_sum_d(qs);
    Q2 = kp.Q2_fixed + block_sum_d(qq);
  } else {
    __syncthreads();
  }
  // closing half kick, frames, TI accumulation, divergence
  double kel = 0.0;
  const bool frame = (m % kp.nstout) == 0 && (mode == 1 || (m == 0 && d.frame_total[r] == 0));
  long long fslot = 0;
  if (frame) fslot = d.frame_total[r] % kp.fcap;
  // the next step's opening is fused into this loop when no block-wide quantity needs the
  // closed state first (Bussi's kinetic energy, DBO's protonation class of lambda_t)
  const bool fuse_open = mode == 1 && dyn && m != end && !kp.bussi && !kp.dbo_on;
  for (int c = threadIdx.x; c < kp.C; c += blockDim.x) {
    const size_t ix = (size_t)r * kp.C + c;
    const double dv = d.dvdl_coul[ix] + d.dvdl_bias[ix];
    double v = d.lamv[ix];
    const double l = d.lam[ix];
    if (dyn && mode == 1) {
      v += 0.5 * kp.dtd * (-dv) / kp.m_lam;
      d.lamv[ix] = v;
    }
    kel += 0.5 * kp.m_lam * v * v;
    if (frame) {
      const size_t fi = ((size_t)r * kp.fcap + fslot) * kp.C + c;
      d.frames[fi] = (float)l;
      const long long *cw = d.cens + ((size_t)r * kp.G + d.c_group[c]) * 2;
      d.frame_cens[fi] = (m > cw[0] && m <= cw[1]) ? 1 : 0;
    }
    if (kp.dbo_on && dyn && mode == 1) {
      // DBO block statistics of the completed step m (R24)
      double *aw = d.dbo_well + ix * 5;
      aw[0] += 1.0;
      if (l < kp.dbo_near) { aw[1] += 1.0; aw[2] += l; }
      else if (l > 1.0 - kp.dbo_near) { aw[3] += 1.0; aw[4] += l; }
      const int lpc = d.c_lp[c];
      const int cls = (lpc >= 0 && d.lam[(size_t)r * kp.C + lpc] >= 0.5) ? 1 : 0;
      double *ab = d.dbo_bar + ix * 4 + 2 * cls;
      ab[0] += 1.0;
      if (l > kp.dbo_trans_lo && l < kp.dbo_trans_hi) ab[1] += 1.0;
    }
    if (!dyn && mode == 1) d.ti_sum[ix] += d.dvdl_coul[ix];   // <dV_coul/dlambda>
    if (!(fabs(l) <= 10.0) || !isfinite(dv)) atomicOr(&d.flags[FLAG_DIVERGED], 1);
    if (fuse_open) {
      // next step's B A O A with the same force (Langevin; see lambda_open)
      const double h = kp.dtd;
      v += 0.5 * h * (-dv) / kp.m_lam;                                          // B
      double ln = l + 0.5 * h * v;                                              // A
      v = kp.c1_lam * v + kp.sd_lam * lambda_normal(d.seed[r], (uint32_t)m, (uint32_t)c);   // O
      ln += 0.5 * h * v;                                                        // A
      d.lamv[ix] = v;
      d.lam[ix] = ln;
    }
  }
  if (energy) kel = block_sum_d(kel);
  if (threadIdx.x == 0) {
    if (frame) {
      d.frame_step[(size_t)r * kp.fcap + fslot] = m;
      d.frame_label[(size_t)r * kp.fcap + fslot] = kp.P ? d.remd_label[r] : -1;
      d.frame_total[r] += 1;
    }
    if (energy) {
      double *e = d.erec + ((size_t)(m & 1) * kp.R + r) * kNE;
      e[CPH_E_SELF] = -f * kp.beta_d / sqrtpi * Q2;
      e[CPH_E_NET] = -f * kPi * Q * Q / (2.0 * V * kp.beta_d * kp.beta_d);
      e[CPH_E_BIAS] = ebias;
      e[CPH_E_KE_LAMBDA] = dyn ? kel : 0.0;
    }
  }
  __syncthreads();
  if (mode == 1) {
    if (fuse_open) lambda_set_charges(kp, d, r, false);
    else if (dyn && m != end) lambda_open(kp, d, r, m, false);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int t = atomicAdd(d.done_counter, 1);
      if (t == kp.R - 1) {           // last replica CTA: advance the step counter
        *d.step = m;
        *d.done_counter = 0;
        d.flags[FLAG_PENDING_CLOSE] = 1;
        if (!dyn) *d.ti_n += 1;
        __threadfence();
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_lambda_open(KParams kp, DevBufs d) {
  if (kp.mode != 0) return;
  lambda_open(kp, d, blockIdx.x, *d.step);
}

__global__ void __launch_bounds__(256) k_set_charges(KParams kp, DevBufs d) {
  lambda_set_charges(kp, d, blockIdx.x);
}

// ---- launchers ------------------------------------------------------------------------
int launch_integrate(Ctx &c, cudaStream_t s, int) {
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_integrate<<<grid, 128, 0, s>>>(c.kp, c.d);
  if (!c.kp.bussi) return 1;
  k_thermo<<<grid, 128, 0, s>>>(c.kp, c.d);
  return 2;
}
int launch_close(Ctx &c, cudaStream_t s, int kick) {
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_close<<<grid, 128, 0, s>>>(c.kp, c.d, kick);
  return 1;
}
int launch_lambda_reduce(Ctx &c, cudaStream_t s, int mode) {
  const size_t smem = 3 * sizeof(double) * (size_t)c.kp.nlam;
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_lambda_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_lambda_reduce<<<c.kp.R, 256, smem, s>>>(c.kp, c.d, mode);
  return 1;
}
int launch_lambda_open(Ctx &c, cudaStream_t s) {
  k_lambda_open<<<c.kp.R, 256, 0, s>>>(c.kp, c.d);
  return 1;
}
int launch_set_charges(Ctx &c, cudaStream_t s) {
  k_set_charges<<<c.kp.R, 256, 0, s>>>(c.kp, c.d);
  return 1;
}

}  // namespace cph
