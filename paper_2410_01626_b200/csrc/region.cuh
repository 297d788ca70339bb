// Block / region geometry shared by the list builder and the pair kernel.
//
// Cells (edge >= rlist/2) are grouped into blocks of b[0] x b[1] x b[2] cells.  The region
// of a block is every cell within +-2 cells of it (or the whole dimension when the block
// plus the stencil covers it), i.e. every cell any atom of the block can have neighbours
// in.  A CTA stages its region's atoms in shared memory in a canonical order (region cells
// in (a, b, c) order, each cell's atoms in slot order), so list entries can hold 16-bit
// region-local indices and the pair kernel reads neighbours from shared memory instead of
// gathering them through L1.
#pragma once
#include "cph_device.cuh"

namespace cph {

struct Region {
  int o[3];     // region origin cell (may be negative before wrapping)
  int w[3];     // region width in cells
  int b0[3];    // first cell of the block
  int bw[3];    // block width in cells
  int ncells, nbcells;
};

__device__ __forceinline__ Region block_region(const KParams &kp, int blk) {
  Region g;
  int t = blk;
  const int Z = t % kp.nb[2]; t /= kp.nb[2];
  const int Y = t % kp.nb[1];
  const int X = t / kp.nb[1];
  const int B[3] = {X, Y, Z};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g.b0[d] = B[d] * kp.b[d];
    g.bw[d] = min(kp.b[d], kp.nc[d] - g.b0[d]);
    if (kp.ns[d] < 5 || g.bw[d] + 4 >= kp.nc[d]) { g.o[d] = 0; g.w[d] = kp.nc[d]; }
    else { g.o[d] = g.b0[d] - 2; g.w[d] = g.bw[d] + 4; }
  }
  g.ncells = g.w[0] * g.w[1] * g.w[2];
  g.nbcells = g.bw[0] * g.bw[1] * g.bw[2];
  return g;
}

// global cell index of region-local cell lc
__device__ __forceinline__ int region_cell(const KParams &kp, const Region &g, int lc) {
  const int c = lc % g.w[2];
  const int b = (lc / g.w[2]) % g.w[1];
  const int a = lc / (g.w[2] * g.w[1]);
  const int gx = (g.o[0] + a + kp.nc[0]) % kp.nc[0];
  const int gy = (g.o[1] + b + kp.nc[1]) % kp.nc[1];
  const int gz = (g.o[2] + c + kp.nc[2]) % kp.nc[2];
  return (gx * kp.nc[1] + gy) * kp.nc[2] + gz;
}

// region-local cell index of global cell coordinates (gx, gy, gz) (must lie in the region)
__device__ __forceinline__ int region_local(const KParams &kp, const Region &g, int gx, int gy, int gz) {
  const int a = (gx - g.o[0] + 2 * kp.nc[0]) % kp.nc[0];
  const int b = (gy - g.o[1] + 2 * kp.nc[1]) % kp.nc[1];
  const int c = (gz - g.o[2] + 2 * kp.nc[2]) % kp.nc[2];
  return (a * g.w[1] + b) * g.w[2] + c;
}

// Block-wide exclusive scan of the region cells' atom counts into coff[0..ncells] and of
// the block's own cells into ioff[0..nbcells]; all threads must call it.
__device__ inline void region_tables(const KParams &kp, const Region &g, const int *start, int *coff, int *cglob,
                                     int *ioff, int *iglob) {
  __shared__ int s_warp[33];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = (nt + 31) >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    const int n = pass == 0 ? g.ncells : g.nbcells;
    int *off = pass == 0 ? coff : ioff;
    int *glob = pass == 0 ? cglob : iglob;
    int carry = 0;
    for (int base = 0; base < n; base += nt) {
      const int lc = base + tid;
      int cnt = 0;
      if (lc < n) {
        int gc;
        if (pass == 0) gc = region_cell(kp, g, lc);
        else {
          const int c = lc % g.bw[2], b = (lc / g.bw[2]) % g.bw[1], a = lc / (g.bw[2] * g.bw[1]);
          gc = ((g.b0[0] + a) * kp.nc[1] + (g.b0[1] + b)) * kp.nc[2] + (g.b0[2] + c);
        }
        glob[lc] = gc;
        cnt = start[gc + 1] - start[gc];
      }
      int incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_warp[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        int v = lane < nw ? s_warp[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (lane < nw) s_warp[lane] = v;
        if (lane == 31) s_warp[32] = v;
      }
      __syncthreads();
      if (lc < n) off[lc] = carry + incl - cnt + (wid ? s_warp[wid - 1] : 0);
      carry += s_warp[32];
      __syncthreads();
    }
    if (tid == 0) off[n] = carry;
    __syncthreads();
  }
}

// copy the region's atom positions into shared memory (one warp per cell)
__device__ inline void region_stage(const float4 *__restrict__ xq, const int *start, const Region &g,
                                    const int *coff, const int *cglob, float4 *sx, int cap) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  for (int lc = wid; lc < g.ncells; lc += nw) {
    const int gs = start[cglob[lc]];
    const int n = coff[lc + 1] - coff[lc];
    for (int k = lane; k < n; k += 32) {
      const int l = coff[lc] + k;
      if (l < cap) sx[l] = __ldg(xq + gs + k);
    }
  }
}

// i atom t of the block (t < ioff[nbcells]) -> (block cell index, sorted slot)
__device__ __forceinline__ int block_atom_slot(const int *ioff, const int *iglob, const int *start, int nbcells,
                                               int t, int *bc) {
  int lo = 0, hi = nbcells - 1;
  while (lo < hi) {                       // last cell with ioff <= t
    const int mid = (lo + hi + 1) >> 1;
    if (ioff[mid] <= t) lo = mid; else hi = mid - 1;
  }
  *bc = lo;
  return start[iglob[lo]] + (t - ioff[lo]);
}

}  // namespace cph
