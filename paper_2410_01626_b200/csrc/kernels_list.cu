// Spatial sort and Verlet pair list.
//
// Every nstlist steps: atoms are binned into cells of edge >= rlist/2 (stencil +-2, or the
// whole dimension when it has fewer than 5 cells), counting-sorted by cell, ordered by
// original index inside each cell (deterministic layout), and all per-atom arrays are
// permuted.  Then each atom gets a FULL neighbour list (both directions, so the pair kernel
// needs no atomics) of the non-excluded atoms with float32 d^2 < rlist^2, evaluated with the
// canonical round-to-nearest, no-contraction formula of DESIGN.md R14 so that the list is
// bit-exact against the oracle's.  Entries: sorted slot (24 bits) | LJ type (8 bits); stored
// k-major (nbl[k][i]) so a warp reads 128 contiguous bytes per neighbour index.
#include "cph_device.cuh"

namespace cph {

__device__ __forceinline__ int cell_coord(float x, float invL, int nc) {
  const float t = __fmul_rn(x, invL);
  const float s = __fsub_rn(t, floorf(t));
  int c = (int)__fmul_rn(s, (float)nc);
  return c < 0 ? 0 : (c >= nc ? nc - 1 : c);
}

__device__ __forceinline__ int cell_index(const KParams &kp, float4 p) {
  const int cx = cell_coord(p.x, kp.invL[0], kp.nc[0]);
  const int cy = cell_coord(p.y, kp.invL[1], kp.nc[1]);
  const int cz = cell_coord(p.z, kp.invL[2], kp.nc[2]);
  return (cx * kp.nc[1] + cy) * kp.nc[2] + cz;
}

__global__ void k_cell_assign(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + i;
  const int c = cell_index(kp, d.xyzq[idx]);
  d.cell_of[idx] = c;
  d.cell_rank[idx] = atomicAdd(&d.cell_count[(size_t)r * kp.ncell + c], 1);
}

// exclusive scan of the cell counts of one replica (one CTA of 1024 threads per replica)
__global__ void __launch_bounds__(1024) k_cell_scan(KParams kp, DevBufs d) {
  const int r = blockIdx.x;
  const int nc = kp.ncell;
  const int per = (nc + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(nc, b + per);
  const int *cnt = d.cell_count + (size_t)r * nc;
  int *start = d.cell_start + (size_t)r * (nc + 1);
  int s = 0;
  for (int k = b; k < e; ++k) s += cnt[k];
  // block exclusive scan of s
  __shared__ int ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    int v = ws[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += t;
    }
    ws[lane] = v;   // inclusive over warps
  }
  __syncthreads();
  int run = incl - s + (w ? ws[w - 1] : 0);
  for (int k = b; k < e; ++k) { start[k] = run; run += cnt[k]; }
  if (threadIdx.x == blockDim.x - 1) start[nc] = run;
}

__global__ void k_cell_scatter(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + i;
  const int c = d.cell_of[idx];
  const int ns = d.cell_start[(size_t)r * (kp.ncell + 1) + c] + d.cell_rank[idx];
  d.perm_tmp[(size_t)r * kp.Nst + ns] = i;
}

// order each cell's atoms by original index (insertion sort; cells hold ~20-60 atoms)
__global__ void k_cell_sort(KParams kp, DevBufs d) {
  const int r = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= kp.ncell) return;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  int *p = d.perm_tmp + (size_t)r * kp.Nst;
  const int2 *meta = d.meta + (size_t)r * kp.Nst;
  const int b = start[c], e = start[c + 1];
  for (int a = b + 1; a < e; ++a) {
    const int v = p[a];
    const int key = meta[v].x;
    int t = a - 1;
    while (t >= b && meta[p[t]].x > key) { p[t + 1] = p[t]; --t; }
    p[t + 1] = v;
  }
}

__global__ void k_permute(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const size_t base = (size_t)r * kp.Nst;
  const int old = d.perm_tmp[base + i];
  const int2 m = d.meta[base + old];
  // wrap into the home box: list entries then carry each pair's image (kEntryImgShift)
  float4 x = d.xyzq[base + old];
  x.x -= kp.L[0] * floorf(x.x * kp.invL[0]);
  x.y -= kp.L[1] * floorf(x.y * kp.invL[1]);
  x.z -= kp.L[2] * floorf(x.z * kp.invL[2]);
  d.xyzq_alt[base + i] = x;
  d.vel_alt[base + i] = d.vel[base + old];
  d.meta_alt[base + i] = m;
  d.iperm[(size_t)r * kp.N + m.x] = i;
}

__global__ void k_copy_back(KParams kp, DevBufs d) {
  const int r = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + i;
  d.xyzq[idx] = d.xyzq_alt[idx];
  d.vel[idx] = d.vel_alt[idx];
  d.meta[idx] = d.meta_alt[idx];
}

// One warp per cell: the i atoms are the cell's atoms (one per lane, chunks of 32), and every
// stencil cell's atoms are staged through shared memory (coalesced loads, broadcast reads),
// so the loop structure is uniform across the warp.
__global__ void __launch_bounds__(32) k_build_list(KParams kp, DevBufs d) {
  const int r = blockIdx.y, c = blockIdx.x;
  const int lane = threadIdx.x;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  __shared__ float4 sx[32];
  __shared__ int sj[32];
  const int cz = c % kp.nc[2], cy = (c / kp.nc[2]) % kp.nc[1], cx = c / (kp.nc[2] * kp.nc[1]);
  const int ib = start[c], ie = start[c + 1];
  for (int i0 = ib; i0 < ie; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < ie;
    const float4 xi = valid ? xq[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int orig = valid ? meta[i].x : 0;
    const int eb = valid ? d.excl_ptr[orig] : 0, ee = valid ? d.excl_ptr[orig + 1] : 0;
    uint32_t *out = d.nbl + (size_t)r * kp.cap * kp.Nst + (valid ? i : 0);
    int cnt = 0;
    for (int ox = 0; ox < kp.ns[0]; ++ox) {
      const int gx = (cx + kp.so[0] + ox + 2 * kp.nc[0]) % kp.nc[0];
      for (int oy = 0; oy < kp.ns[1]; ++oy) {
        const int gy = (cy + kp.so[1] + oy + 2 * kp.nc[1]) % kp.nc[1];
        for (int oz = 0; oz < kp.ns[2]; ++oz) {
          const int gz = (cz + kp.so[2] + oz + 2 * kp.nc[2]) % kp.nc[2];
          const int cc = (gx * kp.nc[1] + gy) * kp.nc[2] + gz;
          const int jb = start[cc], je = start[cc + 1];
          for (int j0 = jb; j0 < je; j0 += 32) {
            const int nj = min(32, je - j0);
            __syncwarp();
            if (lane < nj) {
              const int j = j0 + lane;
              sx[lane] = xq[j];
              sj[lane] = j | ((meta[j].y & (int)kEntryTypeMask) << kEntryTypeShift);
            }
            __syncwarp();
            if (!valid) continue;
            for (int t = 0; t < nj; ++t) {
              const float4 xj = sx[t];
              // canonical formula (R14): dx = x_j - x_i ; dx -= L rint(dx / L)
              const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
              const float kx = rintf(__fmul_rn(rx, kp.invL[0]));
              const float ky = rintf(__fmul_rn(ry, kp.invL[1]));
              const float kz = rintf(__fmul_rn(rz, kp.invL[2]));
              const float dx = __fsub_rn(rx, __fmul_rn(kp.L[0], kx));
              const float dy = __fsub_rn(ry, __fmul_rn(kp.L[1], ky));
              const float dz = __fsub_rn(rz, __fmul_rn(kp.L[2], kz));
              const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
              const int je_ = sj[t] | ((((int)kx + 1) * 9 + ((int)ky + 1) * 3 + ((int)kz + 1)) << kEntryImgShift);
              const int j = je_ & (int)kEntryJMask;
              if (!(d2 < kp.rlist2) || j == i) continue;
              if (ee > eb) {
                const int oj = meta[j].x;
                bool ex = false;
                for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == oj);
                if (ex) continue;
              }
              if (cnt < kp.cap) out[(size_t)cnt * kp.Nst] = (uint32_t)je_;
              ++cnt;
            }
          }
        }
      }
    }
    if (valid) {
      d.nnb[base + i] = cnt;
      if (cnt > kp.cap) {
        d.flags[FLAG_LIST_OVERFLOW] = 1;
        atomicMax(&d.flags[FLAG_MAX_NNB], cnt);
      }
    }
  }
}

int launch_rebuild(Ctx &c, cudaStream_t s) {
  const KParams &kp = c.kp;
  dim3 ga((kp.N + 127) / 128, kp.R);
  cudaMemsetAsync(c.d.cell_count, 0, sizeof(int) * (size_t)kp.R * kp.ncell, s);
  k_cell_assign<<<ga, 128, 0, s>>>(kp, c.d);
  k_cell_scan<<<kp.R, 1024, 0, s>>>(kp, c.d);
  k_cell_scatter<<<ga, 128, 0, s>>>(kp, c.d);
  k_cell_sort<<<dim3((kp.ncell + 127) / 128, kp.R), 128, 0, s>>>(kp, c.d);
  k_permute<<<ga, 128, 0, s>>>(kp, c.d);
  k_copy_back<<<ga, 128, 0, s>>>(kp, c.d);
  k_build_list<<<dim3(kp.ncell, kp.R), 32, 0, s>>>(kp, c.d);
  return 7;
}

}  // namespace cph
