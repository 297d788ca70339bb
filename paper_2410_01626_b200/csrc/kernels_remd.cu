// pH replica exchange (R29, R30).
//
// Replicas form ladders of P pH levels (global replica g in ladder g / P, label = its level).
// k_remd_energy writes, per local replica, the row (label, E_0 .. E_{P-1}) with E_p the
// pH-dependent bias (VpH + Vdw with level p's PFC depths) at its current lambda.  Rows of all
// contexts are concatenated in global order (one NCCL all-gather across GPUs, or the local
// buffer on one GPU); k_remd_apply then takes every Metropolis decision of the attempt
// (identically on every rank: same rows, same Philox counters), updates the labels of the
// local replicas and copies their new level's dG / d1 rows; k_bias_refresh re-evaluates
// dV_bias/dlambda and the bias energy so the next step starts on the new Hamiltonian.
#include "cph_device.cuh"

namespace cph {

__global__ void __launch_bounds__(128) k_remd_energy(KParams kp, DevBufs d, double *rows) {
  const int r = blockIdx.x;
  const int P = kp.P;
  double *row = rows + (size_t)r * (P + 1);
  if (threadIdx.x == 0) row[0] = (double)d.remd_label[r];
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    double e = 0.0;
    for (int g = 0; g < kp.G; ++g) {
      const int kind = d.g_kind[g], c0 = d.g_cptr[g];
      const size_t ic = (size_t)r * kp.C + c0;
      const double lp = d.lam[ic], lt = kind == 3 ? d.lam[ic + 1] : 0.0;
      double dp, dt;
      e += group_bias_eval(kind, nullptr, d.lvl_dG + ((size_t)p * kp.G + g) * 3, d.lvl_d1 + (size_t)p * kp.C + c0,
                           d.dw + ic * 4, kp.wall_k, lp, lt, &dp, &dt);
    }
    row[1 + p] = e;
  }
}

__global__ void __launch_bounds__(1024) k_remd_apply(KParams kp, DevBufs d, const double *rows, uint64_t seed,
                                                     long long attempt) {
  const int P = kp.P, Rt = kp.remd_total, L = Rt / P;
  const int npair = (P - 1 - (int)(attempt & 1) + 1) / 2;       // pairs p = attempt%2, +2, ... < P-1
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int g = threadIdx.x; g < Rt; g += blockDim.x) d.remd_holder[g] = -1;
  __syncthreads();
  // each ladder must hold every level once: a duplicated label (CAS finds the slot taken) or
  // a missing one (slot still -1 below) makes the attempt a no-op and raises FLAG_REMD_BAD
  for (int g = threadIdx.x; g < Rt; g += blockDim.x) {
    const double lv = rows[(size_t)g * (P + 1)];
    const int lab = (int)lv;
    if (!(lv >= 0.0 && lv < (double)P) || atomicCAS(&d.remd_holder[(g / P) * P + lab], -1, g) != -1) bad = 1;
    d.remd_newlab[g] = lab;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < Rt; g += blockDim.x)
    if (d.remd_holder[g] < 0) bad = 1;
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) d.flags[FLAG_REMD_BAD] = 1;
    return;
  }
  const double beta = 1.0 / kp.kT;
  for (int t = threadIdx.x; t < L * npair; t += blockDim.x) {
    const int l = t / npair, p = (int)(attempt & 1) + 2 * (t % npair);
    const int i = d.remd_holder[l * P + p], j = d.remd_holder[l * P + p + 1];
    const double *Ei = rows + (size_t)i * (P + 1) + 1, *Ej = rows + (size_t)j * (P + 1) + 1;
    const double delta = (Ei[p + 1] + Ej[p] - Ei[p] - Ej[p + 1]) * beta;
    bool acc = true;
    if (delta > 0.0) {
      const U4 o = philox4x32_10(U4{(uint32_t)attempt, (uint32_t)l, (uint32_t)p, 5u}, (uint32_t)seed,
                                 (uint32_t)(seed >> 32));
      const double u = ((double)o.x + 0.5) * 2.3283064365386963e-10;
      acc = u < exp(-delta);
    }
    d.remd_att[l * (P - 1) + p] += 1;
    if (acc) {
      d.remd_acc[l * (P - 1) + p] += 1;
      d.remd_newlab[i] = p + 1;
      d.remd_newlab[j] = p;
    }
  }
  __syncthreads();
  // local replicas: new labels and their level's pH-dependent tables
  const int per = kp.G * 3 + kp.C;
  for (int t = threadIdx.x; t < kp.R * per; t += blockDim.x) {
    const int r = t / per, k = t % per;
    const int lab = d.remd_newlab[kp.remd_first + r];
    if (k < kp.G * 3) d.g_dG[(size_t)r * kp.G * 3 + k] = d.lvl_dG[(size_t)lab * kp.G * 3 + k];
    else d.d1[(size_t)r * kp.C + (k - kp.G * 3)] = d.lvl_d1[(size_t)lab * kp.C + (k - kp.G * 3)];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < kp.R; r += blockDim.x) d.remd_label[r] = d.remd_newlab[kp.remd_first + r];
}

// dV_bias/dlambda and the bias energy of the current step after a change of the
// pH-dependent tables (the Coulomb part is unchanged)
__global__ void __launch_bounds__(128) k_bias_refresh(KParams kp, DevBufs d) {
  const int r = blockIdx.x;
  const long long n = *d.step;
  double e = 0.0;
  for (int g = threadIdx.x; g < kp.G; g += blockDim.x) {
    const int kind = d.g_kind[g], c0 = d.g_cptr[g];
    const size_t ic = (size_t)r * kp.C + c0;
    const double lp = d.lam[ic], lt = kind == 3 ? d.lam[ic + 1] : 0.0;
    double dp, dt;
    e += group_bias_eval(kind, d.vmm + 36 * (size_t)g, d.g_dG + ((size_t)r * kp.G + g) * 3, d.d1 + ic, d.dw + ic * 4,
                         kp.wall_k, lp, lt, &dp, &dt);
    d.dvdl_bias[ic] = dp;
    if (kind == 3) d.dvdl_bias[ic + 1] = dt;
  }
  e = warp_sum_d(e);
  __shared__ double red[4];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0)
    d.erec[((size_t)(n & 1) * kp.R + r) * kNE + CPH_E_BIAS] = red[0] + red[1] + red[2] + red[3];
}

int launch_remd_energy(Ctx &c, cudaStream_t s, double *rows) {
  k_remd_energy<<<c.kp.R, 128, 0, s>>>(c.kp, c.d, rows);
  return 1;
}
int launch_remd_apply(Ctx &c, cudaStream_t s, const double *rows_all, uint64_t seed, long long attempt) {
  k_remd_apply<<<1, 1024, 0, s>>>(c.kp, c.d, rows_all, seed, attempt);
  return 1;
}
int launch_bias_refresh(Ctx &c, cudaStream_t s) {
  k_bias_refresh<<<c.kp.R, 128, 0, s>>>(c.kp, c.d);
  return 1;
}

}  // namespace cph
