// Spatial sort and Verlet pair list.
//
// Every nstlist steps: atoms are binned into cells of edge >= rlist/2 (stencil +-2, or the
// whole dimension when it has fewer than 5 cells), counting-sorted by cell, ordered by
// (z, original index) inside each cell (deterministic layout), positions are wrapped into the
// box, and all per-atom arrays are permuted.  Then each atom gets a FULL neighbour list (both directions, so the pair kernel
// needs no atomics) of the non-excluded atoms with float32 d^2 < rlist^2, evaluated with the
// canonical round-to-nearest, no-contraction formula of DESIGN.md R14 so that the list is
// bit-exact against the oracle's.  Entries: region-local index (16 bits) | LJ type (5 bits) |
// periodic image code (5 bits); stored k-major (nbl[k][i]) so a warp reads 128 contiguous
// bytes per neighbour index.
#include "region.cuh"

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

__device__ __forceinline__ float wrap_coord(float x, float L, float invL) { return x - L * floorf(x * invL); }

// rint for |t| < 1.5 (round half to even): -1, 0 or +1
// (written with selp so the compiler does not route it through an int->float conversion)
__device__ __forceinline__ float rint_unit(float t) {
  float r;
  asm("{\n\t.reg .pred p, q;\n\t.reg .f32 a;\n\t"
      "setp.gt.f32 p, %1, 0f3F000000;\n\t"
      "setp.lt.f32 q, %1, 0fBF000000;\n\t"
      "selp.f32 a, 0f3F800000, 0f00000000, p;\n\t"
      "selp.f32 %0, 0fBF800000, a, q;\n\t}"
      : "=f"(r) : "f"(t));
  return r;
}

// order each cell's atoms by (wrapped z, original index): a deterministic layout in which
// 4 consecutive atoms of a cell form a compact z-slab "cluster" for the list prefilter
// (insertion sort; cells hold ~20-60 atoms)
__global__ void k_cell_sort(KParams kp, DevBufs d) {
  const int r = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= kp.ncell) return;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  int *p = d.perm_tmp + (size_t)r * kp.Nst;
  const int2 *meta = d.meta + (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  const int b = start[c], e = start[c + 1];
  for (int a = b + 1; a < e; ++a) {
    const int v = p[a];
    const float kz = wrap_coord(xq[v].z, kp.L[2], kp.invL[2]);
    const int ko = meta[v].x;
    int t = a - 1;
    while (t >= b) {
      const int w = p[t];
      const float wz = wrap_coord(xq[w].z, kp.L[2], kp.invL[2]);
      if (wz < kz || (wz == kz && meta[w].x < ko)) break;
      p[t + 1] = w;
      --t;
    }
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
  x.x = wrap_coord(x.x, kp.L[0], kp.invL[0]);
  x.y = wrap_coord(x.y, kp.L[1], kp.invL[1]);
  x.z = wrap_coord(x.z, kp.L[2], kp.invL[2]);
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

// One CTA per block: stage the block's region in shared memory, then every thread takes
// i atoms of the block and tests the atoms of its +-2 cell stencil (all in shared memory)
// with the canonical formula.  Entries hold region-local indices (region.cuh).
__global__ void __launch_bounds__(512) k_build_list(KParams kp, DevBufs d) {
  extern __shared__ float4 s_x[];                       // [rcap]
  __shared__ int s_coff[kMaxRegionCells + 1], s_cglob[kMaxRegionCells];
  __shared__ int s_ioff[kMaxBlockCells + 1], s_iglob[kMaxBlockCells];
  const int r = blockIdx.y;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const Region g = block_region(kp, blockIdx.x);
  region_tables(kp, g, start, s_coff, s_cglob, s_ioff, s_iglob);
  const int nreg = s_coff[g.ncells];
  if (threadIdx.x == 0) {
    atomicMax(&d.flags[FLAG_REGION_MAX], nreg);
    if (nreg > kp.rcap) d.flags[FLAG_REGION_OVERFLOW] = 1;
  }
  region_stage(xq, start, g, s_coff, s_cglob, s_x, kp.rcap);
  __syncthreads();
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const float rlist2 = kp.rlist2;
  const int nI = s_ioff[g.nbcells];
  for (int t = threadIdx.x; t < nI; t += blockDim.x) {
    int bc;
    const int i = block_atom_slot(s_ioff, s_iglob, start, g.nbcells, t, &bc);
    const float4 xi = xq[i];
    const int orig = meta[i].x;
    const int eb = d.excl_ptr[orig], ee = d.excl_ptr[orig + 1];
    const int cz = g.b0[2] + bc % g.bw[2];
    const int cy = g.b0[1] + (bc / g.bw[2]) % g.bw[1];
    const int cx = g.b0[0] + bc / (g.bw[2] * g.bw[1]);
    uint32_t *out = d.nbl + (size_t)r * kp.cap * kp.Nst + i;
    const size_t ostride = kp.Nst;
    int cnt = 0;
    for (int ox = 0; ox < kp.ns[0]; ++ox) {
      const int gx = (cx + kp.so[0] + ox + 2 * kp.nc[0]) % kp.nc[0];
      for (int oy = 0; oy < kp.ns[1]; ++oy) {
        const int gy = (cy + kp.so[1] + oy + 2 * kp.nc[1]) % kp.nc[1];
        for (int oz = 0; oz < kp.ns[2]; ++oz) {
          const int gz = (cz + kp.so[2] + oz + 2 * kp.nc[2]) % kp.nc[2];
          const int lc = region_local(kp, g, gx, gy, gz);
          const int jb = s_coff[lc], je = min(s_coff[lc + 1], kp.rcap);
          const int gstart = start[s_cglob[lc]] - jb;       // global slot = local + gstart
          for (int jl = jb; jl < je; ++jl) {
            const float4 xj = s_x[jl];
            // canonical formula (R14): dx = x_j - x_i ; dx -= L rint(dx / L);
            // positions are wrapped into [0, L] at the rebuild, so |dx / L| <= 1 and
            // rint(t) == (t > 0.5) - (t < -0.5) exactly (ties to even)
            const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
            const float kx = rint_unit(__fmul_rn(rx, Linv.x));
            const float ky = rint_unit(__fmul_rn(ry, Linv.y));
            const float kz = rint_unit(__fmul_rn(rz, Linv.z));
            const float dx = __fsub_rn(rx, __fmul_rn(Lbox.x, kx));
            const float dy = __fsub_rn(ry, __fmul_rn(Lbox.y, ky));
            const float dz = __fsub_rn(rz, __fmul_rn(Lbox.z, kz));
            const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
            if (!(d2 < rlist2)) continue;
            const int j = jl + gstart;
            if (j == i) continue;
            const int2 mj = meta[j];
            if (ee > eb) {
              bool ex = false;
              for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == mj.x);
              if (ex) continue;
            }
            const int code = (int)(kx * 9.0f + ky * 3.0f + kz) + 13;
            if (cnt < kp.cap)
              *out = (uint32_t)jl | ((uint32_t)(mj.y & (int)kEntryTypeMask) << kEntryTypeShift) |
                     ((uint32_t)code << kEntryImgShift);
            out += ostride;
            ++cnt;
          }
        }
      }
    }
    d.nnb[base + i] = cnt;
    if (cnt > kp.cap) {
      d.flags[FLAG_LIST_OVERFLOW] = 1;
      atomicMax(&d.flags[FLAG_MAX_NNB], cnt);
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
  const size_t smem = sizeof(float4) * (size_t)kp.rcap;
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaFuncSetAttribute(k_build_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_build_list<<<dim3(kp.nblk, kp.R), kp.bthreads, smem, s>>>(kp, c.d);
  return 7;
}

}  // namespace cph
