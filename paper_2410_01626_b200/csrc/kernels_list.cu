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
  __shared__ float4 sbc[8], sbh[8];    // cluster box centres and half extents
  const int cz = c % kp.nc[2], cy = (c / kp.nc[2]) % kp.nc[1], cx = c / (kp.nc[2] * kp.nc[1]);
  const int ib = start[c], ie = start[c + 1];
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const float rlist2 = kp.rlist2;
  const float rlist2_pre = kp.rlist2 * 1.001f;
  // stencil tables (cell index and, for +-2 stencils, the uniform periodic image shift
  // L * floor(raw / nc) of that j-cell; dimensions with < 5 cells use per-lane images)
  __shared__ int s_cell[3][8];
  __shared__ float s_wsh[3][8];
  if (lane < 24) {
    const int dd = lane >> 3, o = lane & 7;
    const int cdim = dd == 0 ? cx : (dd == 1 ? cy : cz);
    if (o < kp.ns[dd]) {
      const int raw = cdim + kp.so[dd] + o;
      s_cell[dd][o] = (raw + 2 * kp.nc[dd]) % kp.nc[dd];
      s_wsh[dd][o] = kp.ns[dd] == 5 ? kp.L[dd] * (float)((raw + kp.nc[dd]) / kp.nc[dd] - 1) : 0.f;
    }
  }
  __syncwarp();
  for (int i0 = ib; i0 < ie; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < ie;
    const float4 xi = valid ? xq[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int orig = valid ? meta[i].x : 0;
    const int eb = valid ? d.excl_ptr[orig] : 0, ee = valid ? d.excl_ptr[orig + 1] : 0;
    uint32_t *out = d.nbl + (size_t)r * kp.cap * kp.Nst + (valid ? i : 0);
    const size_t ostride = kp.Nst;
    int cnt = 0;
    for (int ox = 0; ox < kp.ns[0]; ++ox) {
      const int gx = s_cell[0][ox];
      const float wsx = s_wsh[0][ox];
      for (int oy = 0; oy < kp.ns[1]; ++oy) {
        const int gy = s_cell[1][oy];
        const float wsy = s_wsh[1][oy];
        for (int oz = 0; oz < kp.ns[2]; ++oz) {
          const int cc = (gx * kp.nc[1] + gy) * kp.nc[2] + s_cell[2][oz];
          const float wsz = s_wsh[2][oz];
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
            // bounding box of each cluster of 4 consecutive staged atoms (z-sorted in the cell)
            {
              float4 p = sx[min(lane, nj - 1)];
              float lo_x = p.x, lo_y = p.y, lo_z = p.z, hi_x = p.x, hi_y = p.y, hi_z = p.z;
#pragma unroll
              for (int o = 1; o < 4; o <<= 1) {
                lo_x = fminf(lo_x, __shfl_xor_sync(0xffffffffu, lo_x, o));
                lo_y = fminf(lo_y, __shfl_xor_sync(0xffffffffu, lo_y, o));
                lo_z = fminf(lo_z, __shfl_xor_sync(0xffffffffu, lo_z, o));
                hi_x = fmaxf(hi_x, __shfl_xor_sync(0xffffffffu, hi_x, o));
                hi_y = fmaxf(hi_y, __shfl_xor_sync(0xffffffffu, hi_y, o));
                hi_z = fmaxf(hi_z, __shfl_xor_sync(0xffffffffu, hi_z, o));
              }
              if ((lane & 3) == 0) {
                sbc[lane >> 2] = make_float4(0.5f * (lo_x + hi_x) + wsx, 0.5f * (lo_y + hi_y) + wsy,
                                             0.5f * (lo_z + hi_z) + wsz, 0.f);
                sbh[lane >> 2] = make_float4(0.5f * (hi_x - lo_x), 0.5f * (hi_y - lo_y), 0.5f * (hi_z - lo_z), 0.f);
              }
              __syncwarp();
            }
            if (!valid) continue;
            // four candidates (one cluster) per pass (ILP); appends stay in candidate order
            for (int t0 = 0; t0 < nj; t0 += 4) {
              // conservative prefilter: distance from x_i to the cluster box (nearest image);
              // the box contains its atoms, so a rejected cluster cannot hold a list pair
              // (margin 1e-3 relative on d^2 covers the float rounding of this estimate)
              {
                const float4 bc = sbc[t0 >> 2], bh = sbh[t0 >> 2];
                float cx_ = bc.x - xi.x, cy_ = bc.y - xi.y, cz_ = bc.z - xi.z;
                if (kp.ns[0] != 5) cx_ -= Lbox.x * rintf(cx_ * Linv.x);
                if (kp.ns[1] != 5) cy_ -= Lbox.y * rintf(cy_ * Linv.y);
                if (kp.ns[2] != 5) cz_ -= Lbox.z * rintf(cz_ * Linv.z);
                const float gx_ = fmaxf(fabsf(cx_) - bh.x, 0.f), gy_ = fmaxf(fabsf(cy_) - bh.y, 0.f),
                            gz_ = fmaxf(fabsf(cz_) - bh.z, 0.f);
                if (gx_ * gx_ + gy_ * gy_ + gz_ * gz_ > rlist2_pre) continue;
              }
              float d2v[4], kxv[4], kyv[4], kzv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float4 xj = sx[min(t0 + u, nj - 1)];
                // canonical formula (R14): dx = x_j - x_i ; dx -= L rint(dx / L)
                const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
                // positions are wrapped into [0, L] at the rebuild, so |dx / L| <= 1 and
                // rint(t) == (t > 0.5) - (t < -0.5) exactly (ties to even); the selects run on
                // the ALU pipe instead of the XU pipe FRND needs
                kxv[u] = rint_unit(__fmul_rn(rx, Linv.x));
                kyv[u] = rint_unit(__fmul_rn(ry, Linv.y));
                kzv[u] = rint_unit(__fmul_rn(rz, Linv.z));
                const float dx = __fsub_rn(rx, __fmul_rn(Lbox.x, kxv[u]));
                const float dy = __fsub_rn(ry, __fmul_rn(Lbox.y, kyv[u]));
                const float dz = __fsub_rn(rz, __fmul_rn(Lbox.z, kzv[u]));
                d2v[u] = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                if (t0 + u >= nj || !(d2v[u] < rlist2)) continue;
                const int code = (int)(kxv[u] * 9.0f + kyv[u] * 3.0f + kzv[u]) + 13;
                const int je_ = sj[t0 + u] | (code << kEntryImgShift);
                const int j = je_ & (int)kEntryJMask;
                if (j == i) continue;
                if (ee > eb) {
                  const int oj = meta[j].x;
                  bool ex = false;
                  for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == oj);
                  if (ex) continue;
                }
                if (cnt < kp.cap) *out = (uint32_t)je_;
                out += ostride;
                ++cnt;
              }
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
