// Smooth PME: order-4 B-spline spread, influence-function solve on the
// R2C half spectrum, potential/force gather.  Grid convention (R16): atom with
// scaled fractional coordinate u = K (x/L - floor(x/L)) puts weight M4(u - k) on grid points
// k = floor(u) - j, j = 0..3 (mod K).  With w = u - floor(u):
//   theta_0 = w^3/6, theta_1 = (-3w^3+3w^2+3w+1)/6, theta_2 = (3w^3-6w^2+4)/6, theta_3 = (1-w)^3/6.
// The FFTs are cuFFT plans (reported as their own line item).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "cph_device.cuh"

namespace cph {

#ifndef CPH_SPREAD_VEC
#define CPH_SPREAD_VEC 1   // float4 reductions along z (A/B switch)
#endif
#ifndef CPH_SPREAD_TPB
#define CPH_SPREAD_TPB 128
#endif
#ifdef CPH_SPREAD_MAXREG
#define SPREAD_ATTR __maxnreg__(CPH_SPREAD_MAXREG)
#else
#define SPREAD_ATTR __launch_bounds__(CPH_SPREAD_TPB)
#endif

__global__ void SPREAD_ATTR k_spread(KParams kp, DevBufs d) {
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
  // the four z points kz-3 .. kz of a row are contiguous unless they wrap; with K_z % 4 == 0
  // they touch one or two aligned float4 blocks, added with vector reductions (REDG.F32x4:
  // 16 or 32 reductions per atom instead of 64)
  const int z0 = kz - 3;
  const bool vec = CPH_SPREAD_VEC && (kp.K[2] & 3) == 0 && z0 >= 0;
  const int a0 = z0 & ~3, off = z0 - a0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int ix = (kx - a + kp.K[0]) % kp.K[0];
    const float qa = p.w * tx[a];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int iy = (ky - b + kp.K[1]) % kp.K[1];
      const float qab = qa * ty[b];
      float *row = g + ((size_t)ix * kp.K[1] + iy) * kp.K[2];
      if (vec) {
        const float v0 = qab * tz[3], v1 = qab * tz[2], v2 = qab * tz[1], v3 = qab * tz[0];   // z0 .. z0+3
        float4 lo, hi;
        lo.x = off == 0 ? v0 : 0.f;
        lo.y = off == 0 ? v1 : (off == 1 ? v0 : 0.f);
        lo.z = off == 0 ? v2 : (off == 1 ? v1 : (off == 2 ? v0 : 0.f));
        lo.w = off == 0 ? v3 : (off == 1 ? v2 : (off == 2 ? v1 : v0));
        hi.x = off == 1 ? v3 : (off == 2 ? v2 : (off == 3 ? v1 : 0.f));
        hi.y = off == 2 ? v3 : (off == 3 ? v2 : 0.f);
        hi.z = off == 3 ? v3 : 0.f;
        hi.w = 0.f;
        atomicAdd(reinterpret_cast<float4 *>(row + a0), lo);
        if (off) atomicAdd(reinterpret_cast<float4 *>(row + a0 + 4), hi);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) atomicAdd(row + iz[c], qab * tz[c]);
      }
    }
  }
}

// Deterministic mode (cph_params.deterministic): the same per-point contributions, converted
// to 64-bit fixed point (2^-40 e) and added with integer atomics, which commute, so the grid is
// bitwise independent of the order in which atoms arrive; k_fx_to_float converts it for the
// FFT and clears the accumulator for the next spread.
constexpr float kFxScale = 1099511627776.0f;          // 2^40
constexpr double kFxInv = 1.0 / 1099511627776.0;

__global__ void __launch_bounds__(128) k_spread_fx(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const float4 p = d.xyzq[(size_t)r * kp.Nst + i];
  if (p.w == 0.0f) return;
  int kx, ky, kz;
  float tx[4], ty[4], tz[4], dd[4];
  bspline4(p.x, kp.invL[0], kp.K[0], kx, tx, dd);
  bspline4(p.y, kp.invL[1], kp.K[1], ky, ty, dd);
  bspline4(p.z, kp.invL[2], kp.K[2], kz, tz, dd);
  unsigned long long *g = d.grid_fx + (size_t)r * kp.K3;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int ix = (kx - a + kp.K[0]) % kp.K[0];
    const float qa = p.w * tx[a];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int iy = (ky - b + kp.K[1]) % kp.K[1];
      const float qab = qa * ty[b];
      unsigned long long *row = g + ((size_t)ix * kp.K[1] + iy) * kp.K[2];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const long long v = __float2ll_rn(qab * tz[c] * kFxScale);
        atomicAdd(row + (kz - c + kp.K[2]) % kp.K[2], (unsigned long long)v);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_fx_to_float(KParams kp, DevBufs d) {
  const size_t n = (size_t)kp.R * kp.K3;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const double v = (double)(long long)d.grid_fx[t] * kFxInv;
    if (kp.fft64) d.grid64[t] = v;
    else d.grid[t] = (float)v;
    d.grid_fx[t] = 0ull;
  }
}

// Small grids (kp.fft64, K^3 <= 32768: tiny test systems and C1): the fp32 spread grid widened
// to fp64 (k_grid_to64), fp64 transforms and solve, and the back-transformed grid rounded once to
// fp32 for the gather and the lambda kernel.  The fp32 transforms' ~3e-7 relative error of E_rec
// otherwise dominates the 1e-6 E_total bar when the total is a small difference of the self,
// reciprocal and real-space terms.
__global__ void __launch_bounds__(256) k_influence64(KParams kp, DevBufs d) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kp.Kc) return;
  const int mz = idx % kp.Kzc;
  const int t = idx / kp.Kzc;
  const int my = t % kp.K[1];
  const int mx = t / kp.K[1];
  const double fx = (double)(mx <= kp.K[0] / 2 ? mx : mx - kp.K[0]) / kp.Ld[0];
  const double fy = (double)(my <= kp.K[1] / 2 ? my : my - kp.K[1]) / kp.Ld[1];
  const double fz = (double)mz / kp.Ld[2];
  const double m2 = fx * fx + fy * fy + fz * fz;
  double G = 0.0;
  if (idx != 0) {
    const double V = kp.Ld[0] * kp.Ld[1] * kp.Ld[2];
    G = exp(-kPi * kPi * m2 / (kp.beta_d * kp.beta_d)) / (kPi * V * m2) * (double)d.bsp[mx] *
        (double)d.bsp[kp.K[0] + my] * (double)d.bsp[kp.K[0] + kp.K[1] + mz];
  }
  d.ginf64[idx] = G;
}

__global__ void __launch_bounds__(256) k_solve64(KParams kp, DevBufs d, int step_offset) {
  const int r = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  double e = 0.0;
  if (idx < kp.Kc) {
    const double G = d.ginf64[idx];
    double2 *cg = d.cgrid64 + (size_t)r * kp.Kc + idx;
    double2 c = *cg;
    if (energy) {
      const int mz = idx % kp.Kzc;
      const double w = (mz == 0 || (2 * mz == kp.K[2])) ? 1.0 : 2.0;
      e = w * G * (c.x * c.x + c.y * c.y);
    }
    c.x *= G;
    c.y *= G;
    *cg = c;
  }
  if (energy) block_atomic_add_d(0.5 * kFCoul * e, d.erec + ((size_t)(m & 1) * kp.R + r) * kNE + CPH_E_RECIP);
}

__global__ void __launch_bounds__(256) k_grid_to32(KParams kp, DevBufs d) {
  const size_t n = (size_t)kp.R * kp.K3;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x)
    d.grid[t] = (float)d.grid64[t];
}

__global__ void __launch_bounds__(256) k_grid_to64(KParams kp, DevBufs d) {
  const size_t n = (size_t)kp.R * kp.K3;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x)
    d.grid64[t] = (double)d.grid[t];
}

int launch_grid_to32(Ctx &c, cudaStream_t s) {
  if (!c.kp.fft64) return 0;
  const size_t n = (size_t)c.kp.R * c.kp.K3;
  k_grid_to32<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(c.kp, c.d);
  return 1;
}

// Influence function G(m) = exp(-pi^2 m^2/beta^2)/(pi V m^2) |b_x|^2 |b_y|^2 |b_z|^2 on the
// R2C half spectrum, G(0) = 0: identical for every replica (one box), so it is tabulated once
// at create and the per-step solve is a streaming multiply.
__global__ void __launch_bounds__(256) k_influence(KParams kp, DevBufs d) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kp.Kc) return;
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
    G = expf(-pi * pi * m2 / (kp.beta * kp.beta)) / (pi * kp.V * m2) * d.bsp[mx] * d.bsp[kp.K[0] + my] *
        d.bsp[kp.K[0] + kp.K[1] + mz];
  }
  d.ginf[idx] = G;
}

// Qhat(m) *= G(m); E_rec = (f/2) sum_m G |Qhat|^2 with interior k_z planes of the half spectrum
// weighted x2 (energy steps only)
__global__ void __launch_bounds__(256) k_solve(KParams kp, DevBufs d, int step_offset) {
  const int r = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const long long m = *d.step + step_offset;
  const bool energy = is_energy_step(m, *d.end_step, kp.nstenergy);
  double e = 0.0;
  if (idx < kp.Kc) {
    const float G = __ldg(d.ginf + idx);
    float2 *cg = d.cgrid + (size_t)r * kp.Kc + idx;
    float2 c = *cg;
    if (energy) {
      const int mz = idx % kp.Kzc;
      const double w = (mz == 0 || (2 * mz == kp.K[2])) ? 1.0 : 2.0;
      e = w * (double)G * ((double)c.x * c.x + (double)c.y * c.y);
    }
    c.x *= G;
    c.y *= G;
    *cg = c;
  }
  if (energy) block_atomic_add_d(0.5 * kFCoul * e, d.erec + ((size_t)(m & 1) * kp.R + r) * kNE + CPH_E_RECIP);
}

int launch_influence(Ctx &c, cudaStream_t s) {
  k_influence<<<(c.kp.Kc + 255) / 256, 256, 0, s>>>(c.kp, c.d);
  if (c.kp.fft64) k_influence64<<<(c.kp.Kc + 255) / 256, 256, 0, s>>>(c.kp, c.d);
  return c.kp.fft64 ? 2 : 1;
}

// forces on every atom (and the fp32 phi_rec reported by cph_get_forces); the fp64 phi_rec of
// the lambda atoms is computed by the lambda kernel itself (pme_phi64), so this kernel runs
// beside it instead of before it
__global__ void __launch_bounds__(128) k_gather(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const float4 p = d.xyzq[(size_t)r * kp.Nst + i];
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
    }
  }
  const float sc = -kp.fcoul * p.w;
  d.f_rec[(size_t)r * kp.Nst + i] = make_float4(sc * gx * (float)kp.K[0] * kp.invL[0], sc * gy * (float)kp.K[1] * kp.invL[1],
                                                sc * gz * (float)kp.K[2] * kp.invL[2], phi);
}

// Brick-staged force gather (A/B alternative, CPH_GATHER=brick; the default is k_gather: at
// C4 x 21 this kernel takes 0.070 ms per step against 0.057, at C5 x 8 0.134 against 0.142 --
// a cell column's brick is ~2.4x its atoms' own xy footprint (3-point halo around 5.5 points),
// so the staged bytes are ~33 floats per atom against 64 L1-hitting reads, and every chunk
// waits for its copies).  One CTA of
// kGbAtoms threads per cell column walks the column's z-sorted atoms kGbAtoms at a time; for
// each chunk the grid region its 4x4x4 stencils cover (the chunk's base-index range per
// dimension + 3, z rounded out to 16-byte blocks) is copied into shared memory with 1-D bulk
// copies (cp.async.bulk, one or two per z row, completion counted on an mbarrier), then every
// atom reads its 64 points from shared memory.  Same arithmetic and order as k_gather (equal to
// rounding: the compiler contracts the two instantiations differently); an atom whose stencil is not inside the brick (it drifted far since
// the rebuild, or the chunk's region exceeds the buffer) reads the global grid instead.
#ifndef CPH_GB_ATOMS
#define CPH_GB_ATOMS 128
#endif
constexpr int kGbAtoms = CPH_GB_ATOMS;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <class F>
__device__ __forceinline__ float4 gather_atom(const KParams &kp, float4 p, int kx, int ky, int kz, const float tx[4],
                                              const float ty[4], const float tz[4], const float dx[4], const float dy[4],
                                              const float dz[4], F val) {
  float phi = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      float s = 0.f, sd = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float v = val(a, b, c);
        s = fmaf(tz[c], v, s);
        sd = fmaf(dz[c], v, sd);
      }
      phi = fmaf(tx[a] * ty[b], s, phi);
      gx = fmaf(dx[a] * ty[b], s, gx);
      gy = fmaf(tx[a] * dy[b], s, gy);
      gz = fmaf(tx[a] * ty[b], sd, gz);
    }
  }
  const float sc = -kp.fcoul * p.w;
  return make_float4(sc * gx * (float)kp.K[0] * kp.invL[0], sc * gy * (float)kp.K[1] * kp.invL[1],
                     sc * gz * (float)kp.K[2] * kp.invL[2], phi);
}

// signed offset of a base index from a reference, in [-K/2, K/2)
__device__ __forceinline__ int wrap_off(int k, int ref, int K) { return ((k - ref + K + K / 2) % K) - K / 2; }

__global__ void __launch_bounds__(kGbAtoms) k_gather_brick(KParams kp, DevBufs d, int cap) {
  extern __shared__ __align__(128) float brick[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ int s_ext[6];
  const int r = blockIdx.y, col = blockIdx.x, t = threadIdx.x;
  const int nz = kp.nc[2];
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const int cs = start[col * nz], ce = start[col * nz + nz];
  const int Kx = kp.K[0], Ky = kp.K[1], Kz = kp.K[2];
  const float *g = d.grid + (size_t)r * kp.K3;
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  float4 *out = d.f_rec + (size_t)r * kp.Nst;
  const int cxi = col / kp.nc[1], cyi = col % kp.nc[1];
  const int refx = (int)(((float)cxi + 0.5f) * (float)Kx / (float)kp.nc[0]) % Kx;
  const int refy = (int)(((float)cyi + 0.5f) * (float)Ky / (float)kp.nc[1]) % Ky;
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  __syncthreads();
  uint32_t phase = 0;
  for (int c0 = cs; c0 < ce; c0 += kGbAtoms) {
    const int i = c0 + t;
    const bool valid = i < ce;
    const float4 p = valid ? xq[i] : xq[c0];
    int kx, ky, kz;
    float tx[4], ty[4], tz[4], dx[4], dy[4], dz[4];
    bspline4(p.x, kp.invL[0], Kx, kx, tx, dx);
    bspline4(p.y, kp.invL[1], Ky, ky, ty, dy);
    bspline4(p.z, kp.invL[2], Kz, kz, tz, dz);
    // the chunk's base-index extents (x, y about the column centre, z about the first atom)
    if (t < 6) s_ext[t] = (t & 1) ? INT_MIN : INT_MAX;
    __syncthreads();
    const int ox = wrap_off(kx, refx, Kx), oy = wrap_off(ky, refy, Ky);
    int rz;
    {
      // one z reference for the whole CTA: the chunk's first atom
      const float4 p0 = xq[c0];
      const float tz0 = p0.z * kp.invL[2];
      rz = (int)floorf((tz0 - floorf(tz0)) * (float)Kz);
      if (rz >= Kz) rz -= Kz;
    }
    const int oz = wrap_off(kz, rz, Kz);
    atomicMin(&s_ext[0], ox); atomicMax(&s_ext[1], ox);
    atomicMin(&s_ext[2], oy); atomicMax(&s_ext[3], oy);
    atomicMin(&s_ext[4], oz); atomicMax(&s_ext[5], oz);
    __syncthreads();
    const int x0 = refx + s_ext[0] - 3, BX = s_ext[1] - s_ext[0] + 4;
    const int y0 = refy + s_ext[2] - 3, BY = s_ext[3] - s_ext[2] + 4;
    const int zlo = rz + s_ext[4] - 3, zhi = rz + s_ext[5];                 // inclusive, unwrapped
    const int z0 = zlo >= 0 ? (zlo & ~3) : -((-zlo + 3) & ~3);                // 16-byte aligned start
    const int BZ = ((zhi + 1 - z0) + 3) & ~3;
    const bool staged = BX * BY * BZ <= cap && BZ <= Kz && BX <= Kx && BY <= Ky;
    if (staged) {
      {
        const int nrow = BX * BY;
        const int zs = ((z0 % Kz) + Kz) % Kz;
        const int n1 = min(BZ, Kz - zs), n2 = BZ - n1;                      // z run and its wrapped part
        if (t == 0) {
          const uint32_t bytes = (uint32_t)(nrow * BZ * 4);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
        }
        __syncthreads();                                   // expect_tx before any copy completes
        for (int q = t; q < nrow; q += kGbAtoms) {
          const int bx = q / BY, by = q % BY;
          const int ix = ((x0 + bx) % Kx + Kx) % Kx, iy = ((y0 + by) % Ky + Ky) % Ky;
          const float *src = g + ((size_t)ix * Ky + iy) * Kz;
          float *dst = brick + (size_t)q * BZ;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(dst)), "l"(src + zs), "r"(n1 * 4), "r"(smem_u32(&bar)) : "memory");
          if (n2 > 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(dst + n1)), "l"(src), "r"(n2 * 4), "r"(smem_u32(&bar)) : "memory");
        }
      }
      // wait for the copies (phase parity)
      asm volatile(
          "{\n\t.reg .pred P1;\n\tLAB_WAIT%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@!P1 bra.uni LAB_WAIT%=;\n\t}" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
      phase ^= 1u;
    }
    if (valid) {
      const int lx = ox - s_ext[0] + 3, ly = oy - s_ext[2] + 3, lz = (rz + oz) - z0;   // local base indices
      float4 f;
      if (staged && lx >= 3 && lx < BX && ly >= 3 && ly < BY && lz >= 3 && lz < BZ) {
        f = gather_atom(kp, p, kx, ky, kz, tx, ty, tz, dx, dy, dz,
                        [&](int a, int b, int c) { return brick[((lx - a) * BY + (ly - b)) * BZ + (lz - c)]; });
      } else {
        f = gather_atom(kp, p, kx, ky, kz, tx, ty, tz, dx, dy, dz, [&](int a, int b, int c) {
          const int ix = (kx - a + Kx) % Kx, iy = (ky - b + Ky) % Ky, iz = (kz - c + Kz) % Kz;
          return __ldg(g + ((size_t)ix * Ky + iy) * Kz + iz);
        });
      }
      out[i] = f;
    }
    __syncthreads();   // the brick is rewritten by the next chunk's copies
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
}

int launch_spread(Ctx &c, cudaStream_t s) {
  if (c.kp.det) {
    k_spread_fx<<<dim3((c.kp.N + 127) / 128, c.kp.R), 128, 0, s>>>(c.kp, c.d);
    const size_t n = (size_t)c.kp.R * c.kp.K3;
    k_fx_to_float<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(c.kp, c.d);
    return 2;
  }
  if (c.kp.fft64) {
    cudaMemsetAsync(c.d.grid, 0, sizeof(float) * (size_t)c.kp.R * c.kp.K3, s);
    k_spread<<<dim3((c.kp.N + CPH_SPREAD_TPB - 1) / CPH_SPREAD_TPB, c.kp.R), CPH_SPREAD_TPB, 0, s>>>(c.kp, c.d);
    const size_t n = (size_t)c.kp.R * c.kp.K3;
    k_grid_to64<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(c.kp, c.d);
    return 2;
  }
  cudaMemsetAsync(c.d.grid, 0, sizeof(float) * (size_t)c.kp.R * c.kp.K3, s);
  dim3 grid((c.kp.N + CPH_SPREAD_TPB - 1) / CPH_SPREAD_TPB, c.kp.R);
  k_spread<<<grid, CPH_SPREAD_TPB, 0, s>>>(c.kp, c.d);
  return 1;
}
int launch_solve(Ctx &c, cudaStream_t s, int step_offset) {
  dim3 grid((c.kp.Kc + 255) / 256, c.kp.R);
  if (c.kp.fft64) k_solve64<<<grid, 256, 0, s>>>(c.kp, c.d, step_offset);
  else k_solve<<<grid, 256, 0, s>>>(c.kp, c.d, step_offset);
  return 1;
}
int launch_gather(Ctx &c, cudaStream_t s) {
  static const bool global = !(getenv("CPH_GATHER") && getenv("CPH_GATHER")[0] == 'b');   // A/B: brick gather
  if (!global && c.kp.K[2] % 4 == 0) {   // 16-byte bulk copies need K_z % 4 == 0
    // brick buffer: the x, y extent of a column (K / n_c + 3 points, plus drift) times the z
    // extent of kGbAtoms atoms at the mean density, with margin; chunks that need more fall back
    const double rho = (double)c.kp.N / ((double)c.kp.Ld[0] * c.kp.Ld[1] * c.kp.Ld[2]);
    const double bx = std::ceil((double)c.kp.K[0] / c.kp.nc[0]) + 5.0, by = std::ceil((double)c.kp.K[1] / c.kp.nc[1]) + 5.0;
    const double zext = kGbAtoms / (rho * (c.kp.Ld[0] / c.kp.nc[0]) * (c.kp.Ld[1] / c.kp.nc[1])) * c.kp.K[2] / c.kp.Ld[2];
    const int cap = (int)std::min(bx * by * (std::ceil(1.5 * zext) + 12.0), 40.0 * 1024 / 4);   // <= 40 KB (static default)
    k_gather_brick<<<dim3(c.kp.nc[0] * c.kp.nc[1], c.kp.R), kGbAtoms, cap * sizeof(float), s>>>(c.kp, c.d, cap);
    return 1;
  }
  dim3 grid((c.kp.N + 127) / 128, c.kp.R);
  k_gather<<<grid, 128, 0, s>>>(c.kp, c.d);
  return 1;
}

}  // namespace cph
