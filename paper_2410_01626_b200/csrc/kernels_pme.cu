// Smooth PME: order-4 B-spline spread, influence-function solve on the
// R2C half spectrum, potential/force gather.  Grid convention (R16): atom with
// scaled fractional coordinate u = K (x/L - floor(x/L)) puts weight M4(u - k) on grid points
// k = floor(u) - j, j = 0..3 (mod K).  With w = u - floor(u):
//   theta_0 = w^3/6, theta_1 = (-3w^3+3w^2+3w+1)/6, theta_2 = (3w^3-6w^2+4)/6, theta_3 = (1-w)^3/6.
// The FFTs are cuFFT plans (reported as their own line item).
#include "cph_device.cuh"

namespace cph {

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

__global__ void __launch_bounds__(128) k_spread(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const float4 p = d.xyzq[(size_t)r * kp.Nst + i];
  if (p.w == 0.0f) return;
  int kx, ky, kz;
  float tx[4], ty[4], tz[4], dd[4];
  bspline4(p.x, kp.invL[0], kp.K[0], kx, tx, dd);
  bspline4(p.y, kp.invL[1], kp.K[1], ky, ty, dd);
  bspline4(p.z, kp.invL[2], kp.K[2], kz, tz, dd);
  float *g = d.grid + (size_t)r * kp.K3;
  int iz[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) iz[c] = (kz - c + kp.K[2]) % kp.K[2];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int ix = (kx - a + kp.K[0]) % kp.K[0];
    const float qa = p.w * tx[a];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int iy = (ky - b + kp.K[1]) % kp.K[1];
      const float qab = qa * ty[b];
      float *row = g + ((size_t)ix * kp.K[1] + iy) * kp.K[2];
#pragma unroll
      for (int c = 0; c < 4; ++c) atomicAdd(row + iz[c], qab * tz[c]);
    }
  }
}

// Qhat(m) *= G(m), G = exp(-pi^2 m^2/beta^2)/(pi V m^2) |b_x|^2 |b_y|^2 |b_z|^2 ; E_rec
__global__ void __launch_bounds__(256) k_solve(KParams kp, DevBufs d, int step_offset) {
  const int r = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  double e = 0.0;
  if (idx < kp.Kc) {
    const int mz = idx % kp.Kzc;
    const int t = idx / kp.Kzc;
    const int my = t % kp.K[1];
    const int mx = t / kp.K[1];
    const float fx = (float)(mx <= kp.K[0] / 2 ? mx : mx - kp.K[0]) * kp.invL[0];
    const float fy = (float)(my <= kp.K[1] / 2 ? my : my - kp.K[1]) * kp.invL[1];
    const float fz = (float)mz * kp.invL[2];
    const float m2 = fx * fx + fy * fy + fz * fz;
    float G = 0.0f;
    if (idx != 0) {
      const float pi = 3.14159265358979f;
      G = expf(-pi * pi * m2 / (kp.beta * kp.beta)) / (pi * kp.V * m2) * d.bsp[mx] *
          d.bsp[kp.K[0] + my] * d.bsp[kp.K[0] + kp.K[1] + mz];
    }
    float2 *cg = d.cgrid + (size_t)r * kp.Kc + idx;
    float2 c = *cg;
    if (energy) {
      const double w = (mz == 0 || (2 * mz == kp.K[2])) ? 1.0 : 2.0;
      e = w * (double)G * ((double)c.x * c.x + (double)c.y * c.y);
    }
    c.x *= G;
    c.y *= G;
    *cg = c;
  }
  if (energy) block_atomic_add_d(0.5 * kFCoul * e, d.erec + ((size_t)(m & 1) * kp.R + r) * kNE + CPH_E_RECIP);
}

template <bool PHI64>
__device__ __forceinline__ void gather_atom(const KParams &kp, const DevBufs &d, int r, int i, bool valid,
                                            float4 p, int lslot) {
  if (!valid) return;
  int kx, ky, kz;
  float tx[4], ty[4], tz[4], dx[4], dy[4], dz[4];
  bspline4(p.x, kp.invL[0], kp.K[0], kx, tx, dx);
  bspline4(p.y, kp.invL[1], kp.K[1], ky, ty, dy);
  bspline4(p.z, kp.invL[2], kp.K[2], kz, tz, dz);
  const float *g = d.grid + (size_t)r * kp.K3;
  int iz[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) iz[c] = (kz - c + kp.K[2]) % kp.K[2];
  float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
  double phid = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int ix = (kx - a + kp.K[0]) % kp.K[0];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int iy = (ky - b + kp.K[1]) % kp.K[1];
      const float *row = g + ((size_t)ix * kp.K[1] + iy) * kp.K[2];
      float s = 0.f, sd = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float v = __ldg(row + iz[c]);
        s = fmaf(tz[c], v, s);
        sd = fmaf(dz[c], v, sd);
      }
      phi = fmaf(tx[a] * ty[b], s, phi);
      gx = fmaf(dx[a] * ty[b], s, gx);
      gy = fmaf(tx[a] * dy[b], s, gy);
      gz = fmaf(tx[a] * ty[b], sd, gz);
      if (PHI64) phid += (double)(tx[a] * ty[b]) * (double)s;
    }
  }
  const float sc = -kp.fcoul * p.w;
  const float4 out = make_float4(sc * gx * (float)kp.K[0] * kp.invL[0], sc * gy * (float)kp.K[1] * kp.invL[1],
                                 sc * gz * (float)kp.K[2] * kp.invL[2], phi);
  d.f_rec[(size_t)r * kp.Nst + i] = out;
  if (PHI64 && lslot >= 0) d.phi64_rec[(size_t)r * kp.nlam + lslot] = phid;
}

__global__ void __launch_bounds__(128) k_gather(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < kp.N;
  const size_t idx = (size_t)r * kp.Nst + (valid ? i : 0);
  const float4 p = d.xyzq[idx];
  const int lslot = valid ? (d.meta[idx].y >> 8) - 1 : -1;
  if (__any_sync(0xffffffffu, lslot >= 0)) gather_atom<true>(kp, d, r, i, valid, p, lslot);
  else gather_atom<false>(kp, d, r, i, valid, p, lslot);
}

int launch_spread(Ctx &c, cudaStream_t s) {
  cudaMemsetAsync(c.d.grid, 0, sizeof(float) * (size_t)c.kp.R * c.kp.K3, s);
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_spread<<<grid, 128, 0, s>>>(c.kp, c.d);
  return 1;
}
int launch_solve(Ctx &c, cudaStream_t s, int step_offset) {
  dim3 grid((c.kp.Kc + 255) / 256, c.kp.R);
  k_solve<<<grid, 256, 0, s>>>(c.kp, c.d, step_offset);
  return 1;
}
int launch_gather(Ctx &c, cudaStream_t s) {
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_gather<<<grid, 128, 0, s>>>(c.kp, c.d);
  return 1;
}

}  // namespace cph
