// Spatial sort and Verlet pair list.
//
// Every nstlist steps: atoms are binned into cells of edge >= rlist/2 (stencil +-2, or the
// whole dimension when it has fewer than 5 cells), counting-sorted by cell, ordered by
// (wrapped z, original index) inside each cell (deterministic layout), and all per-atom
// arrays are permuted.  Then each atom gets a FULL neighbour list (both directions, so the pair kernel
// needs no atomics) of the non-excluded atoms with float32 d^2 < rlist^2, evaluated with the
// canonical round-to-nearest, no-contraction formula of DESIGN.md R14 so that the list is
// bit-exact against the oracle's.  Entries: sorted slot (21 bits) | LJ type (5 bits) | image
// code (5 bits); stored in 8-entry tiles nbl[k/8][i][k%8] so the builder writes whole 32-byte
// sectors per lane and a warp of the pair kernel reads 1 KB contiguous per 8 neighbours.
#include <cstdlib>

#include <type_traits>

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

// the canonical list decision for one pair (R14), used for fast-path candidates
// inside the rounding band
__device__ __forceinline__ bool canonical_in(float4 xj, float4 xi, float3 Lbox, float3 Linv, float rlist2) {
  const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
  const float dx = __fsub_rn(rx, __fmul_rn(Lbox.x, rint_unit(__fmul_rn(rx, Linv.x))));
  const float dy = __fsub_rn(ry, __fmul_rn(Lbox.y, rint_unit(__fmul_rn(ry, Linv.y))));
  const float dz = __fsub_rn(rz, __fmul_rn(Lbox.z, rint_unit(__fmul_rn(rz, Linv.z))));
  return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz)) < rlist2;
}

// one warp per cell: bitonic sort of the 64-bit keys (wrapped z bits, original index) with
// register shuffles for cells of up to 32 atoms; larger cells (rare) fall back to an
// insertion sort by lane 0.  Keys are unique, so the order is deterministic.
__global__ void __launch_bounds__(128) k_cell_sort(KParams kp, DevBufs d) {
  const int r = blockIdx.y, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= kp.ncell) return;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  int *p = d.perm_tmp + (size_t)r * kp.Nst;
  const int2 *meta = d.meta + (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + (size_t)r * kp.Nst;
  const int b = start[c], e = start[c + 1], n = e - b;
  if (n <= 1) return;
  if (n <= 32) {
    unsigned long long key = ~0ull;
    int v = 0;
    if (lane < n) {
      v = p[b + lane];
      const float zw = wrap_coord(xq[v].z, kp.L[2], kp.invL[2]);     // >= 0: bits order like values
      key = ((unsigned long long)__float_as_uint(zw) << 32) | (uint32_t)meta[v].x;
    }
    for (int k = 2; k <= 32; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, j);
        const int ov = __shfl_xor_sync(0xffffffffu, v, j);
        const bool lower = (lane & j) == 0, up = (lane & k) == 0;
        const bool take = lower == up ? other < key : other > key;   // keep min on the low side
        if (take) { key = other; v = ov; }
      }
    if (lane < n) p[b + lane] = v;
    return;
  }
  if (lane) return;
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
// Fast-path (5x5x5) stencil walk: columns by ring around the i-cell's column, cells of a
// column centre-out, so the far cells - whose pairs mostly end up beyond r_c - form the tail
// of every atom's list and the pair kernel's warps skip their Ewald block together.
__constant__ int c_walk[125] = {62, 61, 63, 60, 64, 37, 36, 38, 35, 39, 57, 56, 58, 55, 59, 67, 66, 68, 65, 69, 87, 86, 88, 85, 89, 32, 31, 33, 30, 34, 42, 41, 43, 40, 44, 82, 81, 83, 80, 84, 92, 91, 93, 90, 94, 12, 11, 13, 10, 14, 52, 51, 53, 50, 54, 72, 71, 73, 70, 74, 112, 111, 113, 110, 114, 7, 6, 8, 5, 9, 17, 16, 18, 15, 19, 27, 26, 28, 25, 29, 47, 46, 48, 45, 49, 77, 76, 78, 75, 79, 97, 96, 98, 95, 99, 107, 106, 108, 105, 109, 117, 116, 118, 115, 119, 2, 1, 3, 0, 4, 22, 21, 23, 20, 24, 102, 101, 103, 100, 104, 122, 121, 123, 120, 124};

// padding of the geometric cell bounds and of the z-window radius (nm): >> the fp32
// rounding of wrapped positions (|x| <= L ~ 14 nm, ulp ~ 1e-6)
constexpr float kWinPad = 1e-4f;

__global__ void __launch_bounds__(32) k_build_list(KParams kp, DevBufs d) {
  const int r = blockIdx.y, c = blockIdx.x;
  const int lane = threadIdx.x;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  __shared__ float4 sx[32];
  __shared__ int sj[32];
  __shared__ uint32_t s_buf[16][32];
  const int cz = c % kp.nc[2], cy = (c / kp.nc[2]) % kp.nc[1], cx = c / (kp.nc[2] * kp.nc[1]);
  const int ib = start[c], ie = start[c + 1];
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const float rlist2 = kp.rlist2;
  // band around r_list^2 inside which the fast (image-staged, rounding-different) d^2 may
  // disagree with the canonical fp32 value; |delta d^2| < 1e-5 r_list^2 (R14)
  const float lo2 = kp.rlist2 * (1.0f - 3e-5f), hi2 = kp.rlist2 * (1.0f + 3e-5f);
  const bool fast = kp.ns[0] == 5 && kp.ns[1] == 5 && kp.ns[2] == 5;
  const float csx = kp.L[0] / (float)kp.nc[0], csy = kp.L[1] / (float)kp.nc[1], csz = kp.L[2] / (float)kp.nc[2];
  const float win_r = sqrtf(kp.rlist2) * 1.0001f + kWinPad;
  const float win_r2 = win_r * win_r;
  // stencil tables (cell index and, for +-2 stencils, the uniform periodic image shift
  // L * floor(raw / nc) of that j-cell; dimensions with < 5 cells use per-lane images)
  __shared__ int s_cell[3][8];
  __shared__ float s_wsh[3][8];
  __shared__ int s_wi[3][8];
  if (lane < 24) {
    const int dd = lane >> 3, o = lane & 7;
    const int cdim = dd == 0 ? cx : (dd == 1 ? cy : cz);
    if (o < kp.ns[dd]) {
      const int raw = cdim + kp.so[dd] + o;
      const int w = kp.ns[dd] == 5 ? (raw + kp.nc[dd]) / kp.nc[dd] - 1 : 0;
      s_cell[dd][o] = (raw + 2 * kp.nc[dd]) % kp.nc[dd];
      s_wi[dd][o] = w;
      s_wsh[dd][o] = kp.L[dd] * (float)w;
    }
  }
  __syncwarp();
  // [start, end) of every stencil cell, in the walk order (ox, oy, oz)
  __shared__ int s_jb[125], s_je[125];
  {
    const int nyz = kp.ns[1] * kp.ns[2], nst = kp.ns[0] * nyz;
    for (int t = lane; t < nst; t += 32) {
      const int w = fast ? c_walk[t] : t;
      const int ox = w / nyz, oy = (w / kp.ns[2]) % kp.ns[1], oz = w % kp.ns[2];
      const int cc = (s_cell[0][ox] * kp.nc[1] + s_cell[1][oy]) * kp.nc[2] + s_cell[2][oz];
      s_jb[t] = start[cc];
      s_je[t] = start[cc + 1];
    }
  }
  __syncwarp();
  for (int i0 = ib; i0 < ie; i0 += 32) {
    const int i = i0 + lane;
    const bool valid = i < ie;
    const float4 xi = valid ? xq[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int orig = valid ? meta[i].x : 0;
    const int eb = valid ? d.excl_ptr[orig] : 0, ee = valid ? d.excl_ptr[orig + 1] : 0;
    // list tile layout: entries k of atom i at nbl[r][k / 8][i][k % 8]; each lane
    // collects 8 entries in its shared-memory column and writes them as one 32-byte sector
    uint4 *out = reinterpret_cast<uint4 *>(d.nbl + (size_t)r * kp.cap * kp.Nst) + 2 * (size_t)(valid ? i : 0);
    const size_t ostride = 2 * (size_t)kp.Nst;                 // uint4 per 8-entry block row
    int cnt = 0, flushed = 0;
    // Flat walk over the stencil cells (ox, oy, oz).  Cell ranges come from shared memory
    // and the next cell's first chunk of positions is loaded while the current one is
    // tested, so the warp waits for one memory latency per rebuild instead of two per cell.
    const int nyz = kp.ns[1] * kp.ns[2], nst = kp.ns[0] * nyz;
    float4 pc = make_float4(0.f, 0.f, 0.f, 0.f);
    int tc = 0;
    {
      const int jb = s_jb[0];
      if (lane < s_je[0] - jb) { pc = xq[jb + lane]; tc = meta[jb + lane].y; }
    }
    float zlo = -INFINITY, zhi = INFINITY;
    for (int t = 0; t < nst; ++t) {
      float4 pn = make_float4(0.f, 0.f, 0.f, 0.f);
      int tn = 0;
      if (t + 1 < nst) {
        const int jb = s_jb[t + 1];
        if (lane < s_je[t + 1] - jb) { pn = xq[jb + lane]; tn = meta[jb + lane].y; }
      }
      const int w = fast ? c_walk[t] : t;
      const int ox = w / nyz, oy = (w / kp.ns[2]) % kp.ns[1], oz = w % kp.ns[2];
      const float wsx = s_wsh[0][ox], wsy = s_wsh[1][oy], wsz = s_wsh[2][oz];
      bool skip = false;
      if (fast) {
        if (t % 5 == 0) {                // first cell of a column in the walk
          // z window of this stencil column.  Each lane's reach in z is sqrt(R^2 - dxy^2), dxy
          // its xy distance to the column (geometric cell bounds in the staged image frame,
          // padded); the warp tests only the staged atoms whose z lies in the union of the
          // lanes' windows (cells are z-sorted, so that is a contiguous slice).  R and the pads
          // are far outside the fp32 rounding of d^2, so no accepted pair is cut.
          const float xlo = (float)(cx - 2 + ox) * csx - kWinPad, xhi = xlo + csx + 2.f * kWinPad;
          const float ylo = (float)(cy - 2 + oy) * csy - kWinPad, yhi = ylo + csy + 2.f * kWinPad;
          const float ddx = fmaxf(0.f, fmaxf(xlo - xi.x, xi.x - xhi));
          const float ddy = fmaxf(0.f, fmaxf(ylo - xi.y, xi.y - yhi));
          const float rr2 = win_r2 - ddx * ddx - ddy * ddy;
          zlo = INFINITY; zhi = -INFINITY;
          if (valid && rr2 > 0.f) {
            const float rr = sqrtf(rr2);
            zlo = xi.z - rr; zhi = xi.z + rr;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
            zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
          }
        }
        const float zc = (float)(cz - 2 + oz) * csz;
        skip = !(zlo <= zhi) || zhi < zc - kWinPad || zlo > zc + csz + kWinPad;
      }
      // accepted pairs' canonical image k = -(j-cell shift) (nearest image, r < L/2)
      const int fast_code = (1 - s_wi[0][ox]) * 9 + (1 - s_wi[1][oy]) * 3 + (1 - s_wi[2][oz]);
      const int jb = s_jb[t], je = s_je[t];
      for (int j0 = jb; !skip && j0 < je; j0 += 32) {
        const int nj = min(32, je - j0);
        int tb = 0, te = nj;
        float4 p = pc;
        int ty = tc;
        if (j0 != jb && lane < nj) { p = xq[j0 + lane]; ty = meta[j0 + lane].y; }   // cells > 32 atoms
        __syncwarp();
        {
          float zt = 0.f;
          if (lane < nj) {
            // fast path: stage the j-cell's periodic image (uniform for a +-2 stencil)
            sx[lane] = fast ? make_float4(p.x + wsx, p.y + wsy, p.z + wsz, 0.f) : p;
            sj[lane] = (j0 + lane) | ((ty & (int)kEntryTypeMask) << kEntryTypeShift);
            zt = p.z + wsz;
          }
          if (fast) {
            tb = __popc(__ballot_sync(0xffffffffu, lane < nj && zt < zlo));
            te = __popc(__ballot_sync(0xffffffffu, lane < nj && zt <= zhi));
          }
        }
        __syncwarp();
        if (!valid) continue;
        for (int t0 = tb; t0 < te; t0 += 4) {
          float d2v[4], kxv[4], kyv[4], kzv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 xj = sx[min(t0 + u, te - 1)];
            if (fast) {
              // approximate d^2 from the staged image; exact canonical decision below
              // only for the rare candidates within the rounding band of r_list^2
              const float dx = xj.x - xi.x, dy = xj.y - xi.y, dz = xj.z - xi.z;
              d2v[u] = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));   // within the band
            } else {
              // canonical formula (R14): dx = x_j - x_i ; dx -= L rint(dx / L);
              // positions are wrapped into [0, L] at the rebuild, so |dx / L| <= 1 and
              // rint(t) == (t > 0.5) - (t < -0.5) exactly (ties to even)
              const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
              kxv[u] = rint_unit(__fmul_rn(rx, Linv.x));
              kyv[u] = rint_unit(__fmul_rn(ry, Linv.y));
              kzv[u] = rint_unit(__fmul_rn(rz, Linv.z));
              const float dx = __fsub_rn(rx, __fmul_rn(Lbox.x, kxv[u]));
              const float dy = __fsub_rn(ry, __fmul_rn(Lbox.y, kyv[u]));
              const float dz = __fsub_rn(rz, __fmul_rn(Lbox.z, kzv[u]));
              d2v[u] = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
            }
          }
          // each lane appends accepted entries to its 16-entry shared-memory ring and writes a
          // full 8-entry tile (one 32-byte sector) at most once per 4 candidates
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (t0 + u >= te) continue;
            int code;
            if (fast) {
              if (d2v[u] >= hi2) continue;
              if (d2v[u] >= lo2 && !canonical_in(xq[sj[t0 + u] & (int)kEntryJMask], xi, Lbox, Linv, rlist2)) continue;
              code = fast_code;
            } else {
              if (!(d2v[u] < rlist2)) continue;
              code = (int)(kxv[u] * 9.0f + kyv[u] * 3.0f + kzv[u]) + 13;
            }
            const int je_ = sj[t0 + u] | (code << kEntryImgShift);
            const int j = je_ & (int)kEntryJMask;
            if (j == i) continue;
            if (ee > eb) {                    // solute atoms only
              const int oj = meta[j].x;
              bool ex = false;
              for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == oj);
              if (ex) continue;
            }
            s_buf[cnt & 15][lane] = (uint32_t)je_;
            ++cnt;
          }
          if (cnt - flushed >= 8) {
            if (flushed < kp.cap) {
              const int h = flushed & 8;
              out[0] = make_uint4(s_buf[h][lane], s_buf[h + 1][lane], s_buf[h + 2][lane], s_buf[h + 3][lane]);
              out[1] = make_uint4(s_buf[h + 4][lane], s_buf[h + 5][lane], s_buf[h + 6][lane], s_buf[h + 7][lane]);
              out += ostride;
            }
            flushed += 8;
          }
        }
      }
      pc = pn;
      tc = tn;
    }
    if (valid && cnt > flushed && flushed < kp.cap) {
      // pad the last tile with the atom's own slot at image kPadCode (a box diagonal away: r > r_c, skipped)
      const uint32_t self = (uint32_t)i | ((uint32_t)(meta[i].y & (int)kEntryTypeMask) << kEntryTypeShift) |
                            (kPadCode << kEntryImgShift);
      const int h = flushed & 8;
      for (int k = cnt - flushed; k < 8; ++k) s_buf[h + k][lane] = self;
      out[0] = make_uint4(s_buf[h][lane], s_buf[h + 1][lane], s_buf[h + 2][lane], s_buf[h + 3][lane]);
      out[1] = make_uint4(s_buf[h + 4][lane], s_buf[h + 5][lane], s_buf[h + 6][lane], s_buf[h + 7][lane]);
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

// the canonical decision plus the canonical image code (kx+1)*9 + (ky+1)*3 + (kz+1)
__device__ __forceinline__ bool canonical_in_code(float4 xj, float4 xi, float3 Lbox, float3 Linv, float rlist2,
                                                  int *code) {
  const float rx = __fsub_rn(xj.x, xi.x), ry = __fsub_rn(xj.y, xi.y), rz = __fsub_rn(xj.z, xi.z);
  const float kx = rint_unit(__fmul_rn(rx, Linv.x)), ky = rint_unit(__fmul_rn(ry, Linv.y)),
              kz = rint_unit(__fmul_rn(rz, Linv.z));
  const float dx = __fsub_rn(rx, __fmul_rn(Lbox.x, kx));
  const float dy = __fsub_rn(ry, __fmul_rn(Lbox.y, ky));
  const float dz = __fsub_rn(rz, __fmul_rn(Lbox.z, kz));
  *code = ((int)kx + 1) * 9 + ((int)ky + 1) * 3 + ((int)kz + 1);
  return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz)) < rlist2;
}

// Column builder (default).  A cell column (fixed x, y cells, all z cells) is one contiguous,
// z-sorted slot run, so its atoms are taken 32 consecutive atoms per warp (one i atom per lane,
// ~91 % of the lanes busy against ~56 % for one warp per cell).  For each of the 25 stencil
// columns (raw xy offsets -2..2 with their uniform periodic images) the warp's union z window
// [min(z_i - R_i), max(z_i + R_i)], R_i = sqrt(r_list'^2 - d_xy,i^2), selects the column's
// cells (plus the image run when the window crosses z = 0 or L); their atoms are staged 32 at
// a time in shared memory (structure of arrays, image shift applied) and each lane tests them
// four at a time: the fast d^2 with paired FP32 ops (FADD2 / FMUL2 / FFMA2: the roundings of
// the scalar formula), one warp-level test for a candidate inside the rounding band of
// r_list^2 (those get the exact canonical decision, R14, image included), and
// predicated appends to the lane's 16-entry shared-memory ring in candidate order, flushed as
// whole 32-byte list tiles.  Warps holding an atom with excluded pairs run the same loop with
// the exclusion test compiled in.  (A 64-entry ring flushed once per staged chunk needed 64 KB
// of shared memory per CTA, which shrank the L1 of the pair kernels co-running from other
// replica sub-batches: step +10 %.)
// warps per column CTA: 8, or 4 when the mean column holds at most 160 atoms (C1, C2: 94 and 143
// atoms per column leave half of 8 warps idle; measured C2 x 17 rebuild 0.85 -> 0.71 ms, no change
// at C4, 16 warps much slower); CPH_COL_WARPS=4|8 forces one
constexpr int kStage = 36;      // staged candidates per warp: 32 + sentinel padding for aligned groups of 4
constexpr int kRing = 16;       // per-lane ring: <= 4 accepted per group + 7 pending

template <int kColWarps>
__global__ void __launch_bounds__(32 * kColWarps) k_build_list_col(KParams kp, DevBufs d) {
  const int r = blockIdx.y, colid = blockIdx.x;
  const int cx = colid / kp.nc[1], cy = colid % kp.nc[1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const int nz = kp.nc[2];
  const int cb = start[colid * nz], ce = start[colid * nz + nz];
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const float rlist2 = kp.rlist2;
  const float lo2 = kp.rlist2 * (1.0f - 3e-5f), hi2 = kp.rlist2 * (1.0f + 3e-5f);
  // conservative band test |d^2 - mid| <= hw (a superset of [lo2, hi2): the margin covers the
  // rounding of d^2 - mid); non-band candidates are accepted iff d^2 < lo2, as in the band rule
  const float2 nmid = make_float2(-0.5f * (lo2 + hi2), -0.5f * (lo2 + hi2));
  const float hw = 0.5f * (hi2 - lo2) * 1.01f;
  const float csx = kp.L[0] / (float)kp.nc[0], csy = kp.L[1] / (float)kp.nc[1], csz = kp.L[2] / (float)nz;
  const float win_r = sqrtf(kp.rlist2) * 1.0001f + kWinPad;
  const float win_r2 = win_r * win_r;
  __shared__ int s_colc[25], s_code[25];
  __shared__ float s_sx[25], s_sy[25], s_xlo[25], s_ylo[25];
  // staged candidates, structure of arrays (float2 pairs feed the paired FP32 ops), padded to
  // 36 with far-away sentinels so groups of 4 never need an index clamp
  __shared__ __align__(16) float s_px[kColWarps][kStage], s_py[kColWarps][kStage], s_pz[kColWarps][kStage];
  __shared__ __align__(16) int s_ent[kColWarps][kStage];
  __shared__ int s_org[kColWarps][kStage];
  __shared__ uint32_t s_ring[kColWarps * kRing * 32];
  if (threadIdx.x < 25) {
    const int k = c_walk[threadIdx.x * 5] / 5;            // column ring order around the centre
    const int rx = cx - 2 + k / 5, ry = cy - 2 + k % 5;
    const int wx = (rx + 2 * kp.nc[0]) / kp.nc[0] - 2, wy = (ry + 2 * kp.nc[1]) / kp.nc[1] - 2;
    s_colc[threadIdx.x] = ((rx - wx * kp.nc[0]) * kp.nc[1] + (ry - wy * kp.nc[1])) * nz;
    s_sx[threadIdx.x] = kp.L[0] * (float)wx;
    s_sy[threadIdx.x] = kp.L[1] * (float)wy;
    s_xlo[threadIdx.x] = (float)rx * csx - kWinPad;
    s_ylo[threadIdx.x] = (float)ry * csy - kWinPad;
    s_code[threadIdx.x] = (1 - wx) * 9 + (1 - wy) * 3;
  }
  __syncthreads();
  float *px = s_px[w], *py = s_py[w], *pz = s_pz[w];
  int *sj = s_ent[w], *so = s_org[w];
  if (lane < kStage - 32) {
    px[32 + lane] = py[32 + lane] = pz[32 + lane] = 1e30f;
    sj[32 + lane] = 0;
    so[32 + lane] = -1;
  }
  uint32_t *ring = s_ring + w * kRing * 32 + lane;      // entry k at ring[(k & 15) * 32]
  uint32_t *nbl = d.nbl + (size_t)r * kp.cap * kp.Nst;
  for (int i0 = cb + 32 * w; i0 < ce; i0 += 32 * kColWarps) {
    const int i = i0 + lane;
    const bool valid = i < ce;
    const float4 xi = valid ? xq[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int orig = valid ? meta[i].x : 0;
    const int eb = valid ? d.excl_ptr[orig] : 0, ee = valid ? d.excl_ptr[orig + 1] : 0;
    const bool warp_excl = __any_sync(0xffffffffu, ee > eb);
    const float2 nxi = make_float2(-xi.x, -xi.x), nyi = make_float2(-xi.y, -xi.y), nzi = make_float2(-xi.z, -xi.z);
    uint4 *out = reinterpret_cast<uint4 *>(nbl) + 2 * (size_t)(valid ? i : 0);
    const size_t ostride = 2 * (size_t)kp.Nst;
    int cnt = 0, flushed = 0;
    auto excluded = [&](int oj) {
      bool ex = false;
      for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == oj);
      return ex;
    };
    // test the staged slice [tb, te) four candidates at a time (EXCL: exclusion test compiled in)
    auto scan = [&](auto excl_tag, int tb, int te, int tself, int fast_code) {
      constexpr bool EXCL = decltype(excl_tag)::value;
      for (int t0 = tb & ~3; t0 < te; t0 += 4) {
        const float4 x4 = *reinterpret_cast<const float4 *>(px + t0);
        const float4 y4 = *reinterpret_cast<const float4 *>(py + t0);
        const float4 z4 = *reinterpret_cast<const float4 *>(pz + t0);
        const int4 e4 = *reinterpret_cast<const int4 *>(sj + t0);
        const int ev[4] = {e4.x, e4.y, e4.z, e4.w};
        const float2 xa = make_float2(x4.x, x4.y), xb = make_float2(x4.z, x4.w);
        const float2 ya = make_float2(y4.x, y4.y), yb = make_float2(y4.z, y4.w);
        const float2 za = make_float2(z4.x, z4.y), zb = make_float2(z4.z, z4.w);
        const float2 dxa = __fadd2_rn(xa, nxi), dxb = __fadd2_rn(xb, nxi);
        const float2 dya = __fadd2_rn(ya, nyi), dyb = __fadd2_rn(yb, nyi);
        const float2 dza = __fadd2_rn(za, nzi), dzb = __fadd2_rn(zb, nzi);
        const float2 qa = __ffma2_rn(dxa, dxa, __ffma2_rn(dya, dya, __fmul2_rn(dza, dza)));
        const float2 qb = __ffma2_rn(dxb, dxb, __ffma2_rn(dyb, dyb, __fmul2_rn(dzb, dzb)));
        const float2 ma = __fadd2_rn(qa, nmid), mb = __fadd2_rn(qb, nmid);
        const float d2[4] = {qa.x, qa.y, qb.x, qb.y};
        if (!(fminf(fminf(fabsf(ma.x), fabsf(ma.y)), fminf(fabsf(mb.x), fabsf(mb.y))) <= hw)) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            bool ok = d2[u] < lo2 && t0 + u != tself;
            if (EXCL && ok && ee > eb) ok = !excluded(so[t0 + u]);
            if (ok) {
              ring[(cnt & (kRing - 1)) * 32] = (uint32_t)ev[u];
              ++cnt;
            }
          }
        } else {                                 // rare: a candidate near r_list^2
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (!(d2[u] < hi2)) continue;
            const int je = ev[u];
            const int j = je & (int)kEntryJMask;
            if (!(d2[u] < lo2)) {
              int cc;
              if (!canonical_in_code(xq[j], xi, Lbox, Linv, rlist2, &cc) || cc != fast_code) continue;
            }
            if (j == i) continue;
            if (EXCL && ee > eb && excluded(so[t0 + u])) continue;
            ring[(cnt & (kRing - 1)) * 32] = (uint32_t)je;
            ++cnt;
          }
        }
        if (cnt - flushed >= 8) {                // flush a whole 32-byte tile
          if (flushed < kp.cap) {
            const uint32_t *t = ring + (flushed & (kRing - 1)) * 32;
            out[0] = make_uint4(t[0], t[32], t[64], t[96]);
            out[1] = make_uint4(t[128], t[160], t[192], t[224]);
            out += ostride;
          }
          flushed += 8;
        }
      }
    };
    for (int q = 0; q < 25; ++q) {
      const float xlo = s_xlo[q], ylo = s_ylo[q];
      const float ddx = fmaxf(0.f, fmaxf(xlo - xi.x, xi.x - (xlo + csx + 2.f * kWinPad)));
      const float ddy = fmaxf(0.f, fmaxf(ylo - xi.y, xi.y - (ylo + csy + 2.f * kWinPad)));
      const float rr2 = win_r2 - ddx * ddx - ddy * ddy;
      float zlo = INFINITY, zhi = -INFINITY;
      if (valid && rr2 > 0.f) {
        const float rr = sqrtf(rr2);
        zlo = xi.z - rr;
        zhi = xi.z + rr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
        zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
      }
      if (!(zlo <= zhi)) continue;
      const int colc = s_colc[q];
      const float wsx = s_sx[q], wsy = s_sy[q];
      // runs: the home z image, the image below 0, the image above L (the union window of
      // a warp in a short box can cross both ends; each lane's own reach R < L/2 never does)
      for (int part = 0; part < 3; ++part) {
        float a, b, wsz;
        int wz;
        if (part == 0) { a = fmaxf(zlo, 0.f); b = fminf(zhi, kp.L[2]); wsz = 0.f; wz = 0; }
        else if (part == 1) {
          if (!(zlo < 0.f)) continue;
          a = zlo + kp.L[2]; b = kp.L[2]; wsz = -kp.L[2]; wz = -1;
        } else {
          if (!(zhi > kp.L[2])) continue;
          a = 0.f; b = zhi - kp.L[2]; wsz = kp.L[2]; wz = 1;
        }
        if (!(a <= b)) continue;
        const int c0 = max(0, min((int)floorf(a / csz), nz - 1));
        const int c1 = max(0, min((int)floorf(b / csz), nz - 1));
        const int j0 = start[colc + c0], j1 = start[colc + c1 + 1];
        const int fast_code = s_code[q] + (1 - wz);
        const float zwlo = zlo - wsz, zwhi = zhi - wsz;      // window in the staged frame's terms
        for (int jb = j0; jb < j1; jb += 32) {
          const int nj = min(32, j1 - jb);
          __syncwarp();
          float zt = 0.f;
          if (lane < nj) {
            const float4 p = xq[jb + lane];
            const int2 mt = meta[jb + lane];
            px[lane] = p.x + wsx;
            py[lane] = p.y + wsy;
            pz[lane] = p.z + wsz;
            sj[lane] = (jb + lane) | ((mt.y & (int)kEntryTypeMask) << kEntryTypeShift) | (fast_code << kEntryImgShift);
            so[lane] = mt.x;
            zt = p.z;
          } else {
            px[lane] = py[lane] = pz[lane] = 1e30f;
          }
          // the staged atoms are z-sorted: the union window is a contiguous slice
          const int tb = __popc(__ballot_sync(0xffffffffu, lane < nj && zt < zwlo));
          const int te = __popc(__ballot_sync(0xffffffffu, lane < nj && zt <= zwhi));
          __syncwarp();
          if (!valid) continue;
          if (warp_excl) scan(std::true_type{}, tb, te, i - jb, fast_code);
          else scan(std::false_type{}, tb, te, i - jb, fast_code);
        }
      }
    }
    if (valid && cnt > flushed && flushed < kp.cap) {
      // pad the last tile with the atom's own slot at image kPadCode (a box diagonal away: r > r_c, skipped)
      const uint32_t self = (uint32_t)i | ((uint32_t)(meta[i].y & (int)kEntryTypeMask) << kEntryTypeShift) |
                            (kPadCode << kEntryImgShift);
      uint32_t *t = ring + (flushed & (kRing - 1)) * 32;
      for (int k = cnt - flushed; k < 8; ++k) t[k * 32] = self;
      out[0] = make_uint4(t[0], t[32], t[64], t[96]);
      out[1] = make_uint4(t[128], t[160], t[192], t[224]);
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

// ---- cluster-pair list (cph_params.pair_list = 2) ------------------------------
// Super-clusters are 32 consecutive atoms of one cell column (column-aligned; the last one of a
// column is partial); super-cluster id = floor(column start / 32) + column index + k, unique
// because column c holds ceil(n_c / 32) <= n_c / 32 + 1 of them.  i-cluster s of a super-cluster
// = its atoms 8s .. 8s+7; j-clusters are globally aligned groups of 4 sorted slots.  For every
// canonical pair (i, j) (R14, not excluded) with slot_i < slot_j, the super-cluster of
// i holds an entry (J = slot_j / 4, image code) whose mask word s has bit (slot_j % 4) * 8 + a,
// a = (slot_i - first) % 8: the bits are exactly the canonical half list.  One warp per
// super-cluster walks the 25 stencil columns like the column builder (union z window of its
// atoms, home and z-image runs), restricted to slots > its first atom, stages 32 slots at a time
// (4-aligned, so a group of 4 staged candidates is one j-cluster) and takes the four per-lane
// decisions of a group with the same fast d^2 / rounding-band / exact canonical test as the
// column builder; four ballots give the group's masks and lane 0 appends the entry.
constexpr int kClWarps = 8;

__global__ void __launch_bounds__(32 * kClWarps, 2) k_build_cluster(KParams kp, DevBufs d) {
  const int r = blockIdx.y, colid = blockIdx.x;
  const int cx = colid / kp.nc[1], cy = colid % kp.nc[1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const int nz = kp.nc[2];
  const int cb = start[colid * nz], ce = start[colid * nz + nz];
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const float rlist2 = kp.rlist2;
  const float lo2 = kp.rlist2 * (1.0f - 3e-5f), hi2 = kp.rlist2 * (1.0f + 3e-5f);
  const float2 nmid = make_float2(-0.5f * (lo2 + hi2), -0.5f * (lo2 + hi2));
  const float hw = 0.5f * (hi2 - lo2) * 1.01f;
  const float csx = kp.L[0] / (float)kp.nc[0], csy = kp.L[1] / (float)kp.nc[1], csz = kp.L[2] / (float)nz;
  const float win_r = sqrtf(kp.rlist2) * 1.0001f + kWinPad;
  const float win_r2 = win_r * win_r;
  __shared__ int s_colc[25], s_code[25];
  __shared__ float s_sx[25], s_sy[25], s_xlo[25], s_ylo[25];
  __shared__ __align__(16) float s_px[kClWarps][32], s_py[kClWarps][32], s_pz[kClWarps][32];
  __shared__ int s_org[kClWarps][32];
  if (threadIdx.x < 25) {
    const int k = c_walk[threadIdx.x * 5] / 5;
    const int rx = cx - 2 + k / 5, ry = cy - 2 + k % 5;
    const int wx = (rx + 2 * kp.nc[0]) / kp.nc[0] - 2, wy = (ry + 2 * kp.nc[1]) / kp.nc[1] - 2;
    s_colc[threadIdx.x] = ((rx - wx * kp.nc[0]) * kp.nc[1] + (ry - wy * kp.nc[1])) * nz;
    s_sx[threadIdx.x] = kp.L[0] * (float)wx;
    s_sy[threadIdx.x] = kp.L[1] * (float)wy;
    s_xlo[threadIdx.x] = (float)rx * csx - kWinPad;
    s_ylo[threadIdx.x] = (float)ry * csy - kWinPad;
    s_code[threadIdx.x] = (1 - wx) * 9 + (1 - wy) * 3;
  }
  __syncthreads();
  float *px = s_px[w], *py = s_py[w], *pz = s_pz[w];
  int *so = s_org[w];
  const int sc0 = cb / kClSuper + colid;
  for (int k = w; kClSuper * k < ce - cb; k += kClWarps) {
    const int first = cb + kClSuper * k, ni = min(kClSuper, ce - first);
    const size_t sidx = (size_t)r * kp.nsc + sc0 + k;
    const int i = first + lane;
    const bool valid = lane < ni;
    const float4 xi = valid ? xq[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int orig = valid ? meta[i].x : 0;
    const int eb = valid ? d.excl_ptr[orig] : 0, ee = valid ? d.excl_ptr[orig + 1] : 0;
    const bool warp_excl = __any_sync(0xffffffffu, ee > eb);
    const float2 nxi = make_float2(-xi.x, -xi.x), nyi = make_float2(-xi.y, -xi.y), nzi = make_float2(-xi.z, -xi.z);
    uint32_t *oj = d.cl_j + sidx * kp.clcap;
    uint4 *om = d.cl_m + sidx * kp.clcap;
    int cnt = 0;
    auto excluded = [&](int o) {
      bool ex = false;
      for (int e = eb; e < ee; ++e) ex |= (d.excl_idx[e] == o);
      return ex;
    };
    for (int q = 0; q < 25; ++q) {
      const float xlo = s_xlo[q], ylo = s_ylo[q];
      const float ddx = fmaxf(0.f, fmaxf(xlo - xi.x, xi.x - (xlo + csx + 2.f * kWinPad)));
      const float ddy = fmaxf(0.f, fmaxf(ylo - xi.y, xi.y - (ylo + csy + 2.f * kWinPad)));
      const float rr2 = win_r2 - ddx * ddx - ddy * ddy;
      float zlo = INFINITY, zhi = -INFINITY;
      if (valid && rr2 > 0.f) {
        const float rr = sqrtf(rr2);
        zlo = xi.z - rr;
        zhi = xi.z + rr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
        zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
      }
      if (!(zlo <= zhi)) continue;
      const int colc = s_colc[q];
      const float wsx = s_sx[q], wsy = s_sy[q];
      for (int part = 0; part < 3; ++part) {
        float a, b, wsz;
        int wz;
        if (part == 0) { a = fmaxf(zlo, 0.f); b = fminf(zhi, kp.L[2]); wsz = 0.f; wz = 0; }
        else if (part == 1) {
          if (!(zlo < 0.f)) continue;
          a = zlo + kp.L[2]; b = kp.L[2]; wsz = -kp.L[2]; wz = -1;
        } else {
          if (!(zhi > kp.L[2])) continue;
          a = 0.f; b = zhi - kp.L[2]; wsz = kp.L[2]; wz = 1;
        }
        if (!(a <= b)) continue;
        const int c0 = max(0, min((int)floorf(a / csz), nz - 1));
        const int c1 = max(0, min((int)floorf(b / csz), nz - 1));
        const int j0 = max(start[colc + c0], first + 1), j1 = start[colc + c1 + 1];   // half list: j > first
        if (j0 >= j1) continue;
        const uint32_t code = (uint32_t)(s_code[q] + (1 - wz));
        const float zwlo = zlo - wsz, zwhi = zhi - wsz;
        for (int jb = j0 & ~3; jb < j1; jb += 32) {
          const int js = jb + lane;
          const bool in = js >= j0 && js < j1;
          __syncwarp();
          float zt = 0.f;
          if (in) {
            const float4 p = xq[js];
            px[lane] = p.x + wsx;
            py[lane] = p.y + wsy;
            pz[lane] = p.z + wsz;
            so[lane] = meta[js].x;
            zt = p.z;
          } else {
            px[lane] = py[lane] = pz[lane] = 1e30f;
            so[lane] = -1;
          }
          // the run [j0, j1) is z-sorted: the union window is a contiguous slice of it
          const int lo_l = max(0, j0 - jb);
          const int tb = lo_l + __popc(__ballot_sync(0xffffffffu, in && zt < zwlo));
          const int te = lo_l + __popc(__ballot_sync(0xffffffffu, in && zt <= zwhi));
          __syncwarp();
          for (int t0 = tb & ~3; t0 < te; t0 += 4) {
            const float4 x4 = *reinterpret_cast<const float4 *>(px + t0);
            const float4 y4 = *reinterpret_cast<const float4 *>(py + t0);
            const float4 z4 = *reinterpret_cast<const float4 *>(pz + t0);
            const float2 dxa = __fadd2_rn(make_float2(x4.x, x4.y), nxi), dxb = __fadd2_rn(make_float2(x4.z, x4.w), nxi);
            const float2 dya = __fadd2_rn(make_float2(y4.x, y4.y), nyi), dyb = __fadd2_rn(make_float2(y4.z, y4.w), nyi);
            const float2 dza = __fadd2_rn(make_float2(z4.x, z4.y), nzi), dzb = __fadd2_rn(make_float2(z4.z, z4.w), nzi);
            const float2 qa = __ffma2_rn(dxa, dxa, __ffma2_rn(dya, dya, __fmul2_rn(dza, dza)));
            const float2 qb = __ffma2_rn(dxb, dxb, __ffma2_rn(dyb, dyb, __fmul2_rn(dzb, dzb)));
            const float2 ma = __fadd2_rn(qa, nmid), mb = __fadd2_rn(qb, nmid);
            const float d2[4] = {qa.x, qa.y, qb.x, qb.y};
            const int jt = jb + t0;                               // slot of candidate u = jt + u
            bool acc[4];
            if (!__any_sync(0xffffffffu, fminf(fminf(fabsf(ma.x), fabsf(ma.y)), fminf(fabsf(mb.x), fabsf(mb.y))) <= hw)) {
#pragma unroll
              for (int u = 0; u < 4; ++u) acc[u] = valid && d2[u] < lo2 && jt + u > i;
            } else {                                              // rare: a candidate near r_list^2
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                bool ok = valid && d2[u] < hi2 && jt + u > i;
                if (ok && !(d2[u] < lo2)) {
                  int cc;
                  ok = canonical_in_code(xq[jt + u], xi, Lbox, Linv, rlist2, &cc) && cc == (int)code;
                }
                acc[u] = ok;
              }
            }
            if (warp_excl) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (acc[u] && ee > eb) acc[u] = !excluded(so[t0 + u]);
            }
            const uint32_t B0 = __ballot_sync(0xffffffffu, acc[0]), B1 = __ballot_sync(0xffffffffu, acc[1]);
            const uint32_t B2 = __ballot_sync(0xffffffffu, acc[2]), B3 = __ballot_sync(0xffffffffu, acc[3]);
            if ((B0 | B1 | B2 | B3) == 0u) continue;
            if (lane == 0) {
              // ballot bit l = 8 s + a  ->  mask word s, bit u * 8 + a
              uint32_t m[4];
#pragma unroll
              for (int s = 0; s < 4; ++s)
                m[s] = ((B0 >> (8 * s)) & 0xFFu) | (((B1 >> (8 * s)) & 0xFFu) << 8) | (((B2 >> (8 * s)) & 0xFFu) << 16) |
                       (((B3 >> (8 * s)) & 0xFFu) << 24);
              if (cnt < kp.clcap) {
                oj[cnt] = (uint32_t)(jt >> 2) | (code << kEntryImgShift);
                om[cnt] = make_uint4(m[0], m[1], m[2], m[3]);
              }
            }
            ++cnt;
          }
        }
      }
    }
    if (lane == 0) {
      d.cl_n[sidx] = cnt;
      d.sc_first[sidx] = first;
      d.sc_ni[sidx] = ni;
      if (cnt > kp.clcap) {
        d.flags[FLAG_CL_OVERFLOW] = 1;
        atomicMax(&d.flags[FLAG_CL_MAX], cnt);
      }
    }
  }
}

// Full canonical rows of the lambda atoms (both directions, slot order per stencil cell) for the
// fp64 real-space potential of the lambda atoms in cluster mode (k_phi_lam): one warp per lambda
// atom, every cell of its 5x5x5 stencil (whole dimensions below 5 cells) visited once, the exact
// canonical decision with the pair's own image code, ballot-compacted in-order appends.
__global__ void __launch_bounds__(32) k_build_lam_list(KParams kp, DevBufs d) {
  const int r = blockIdx.y, k = blockIdx.x, lane = threadIdx.x;
  const size_t base = (size_t)r * kp.Nst;
  const float4 *xq = d.xyzq + base;
  const int2 *meta = d.meta + base;
  const int *start = d.cell_start + (size_t)r * (kp.ncell + 1);
  const int orig = d.g_atoms[k];
  const int i = d.iperm[(size_t)r * kp.N + orig];
  const float4 xi = xq[i];
  const float3 Lbox = make_float3(kp.L[0], kp.L[1], kp.L[2]);
  const float3 Linv = make_float3(kp.invL[0], kp.invL[1], kp.invL[2]);
  const int eb = d.excl_ptr[orig], ee = d.excl_ptr[orig + 1];
  int ci[3];
  {
    const float p[3] = {xi.x, xi.y, xi.z};
    for (int dd = 0; dd < 3; ++dd) ci[dd] = cell_coord(p[dd], kp.invL[dd], kp.nc[dd]);
  }
  uint32_t *out = d.lam_nbl + ((size_t)r * kp.nlam + k) * kp.cap;
  int cnt = 0;
  for (int ox = 0; ox < kp.ns[0]; ++ox)
    for (int oy = 0; oy < kp.ns[1]; ++oy)
      for (int oz = 0; oz < kp.ns[2]; ++oz) {
        const int gx = kp.ns[0] == 5 ? (ci[0] - 2 + ox + kp.nc[0]) % kp.nc[0] : ox;
        const int gy = kp.ns[1] == 5 ? (ci[1] - 2 + oy + kp.nc[1]) % kp.nc[1] : oy;
        const int gz = kp.ns[2] == 5 ? (ci[2] - 2 + oz + kp.nc[2]) % kp.nc[2] : oz;
        const int cc = (gx * kp.nc[1] + gy) * kp.nc[2] + gz;
        const int jb = start[cc], je = start[cc + 1];
        for (int j0 = jb; j0 < je; j0 += 32) {
          const int j = j0 + lane;
          bool ok = false;
          int code = 13;
          if (j < je && j != i) {
            ok = canonical_in_code(xq[j], xi, Lbox, Linv, kp.rlist2, &code);
            if (ok && ee > eb) {
              const int o = meta[j].x;
              for (int e = eb; e < ee; ++e) ok &= (d.excl_idx[e] != o);
            }
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, ok);
          const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
          if (ok && pos < kp.cap) out[pos] = (uint32_t)j | ((uint32_t)code << kEntryImgShift);
          cnt += __popc(bal);
        }
      }
  if (lane == 0) {
    d.lam_n[(size_t)r * kp.nlam + k] = cnt;
    if (cnt > kp.cap) {
      d.flags[FLAG_LIST_OVERFLOW] = 1;
      atomicMax(&d.flags[FLAG_MAX_NNB], cnt);
    }
  }
}

// spatial sort + permutation of every per-atom array (positions wrapped); the pair list
// itself is launch_build_list, so work that only needs the new atom order (the PME chain) can
// start while the list is built
int launch_sort(Ctx &c, cudaStream_t s) {
  const KParams &kp = c.kp;
  dim3 ga((kp.N + 127) / 128, kp.R);
  cudaMemsetAsync(c.d.cell_count, 0, sizeof(int) * (size_t)kp.R * kp.ncell, s);
  k_cell_assign<<<ga, 128, 0, s>>>(kp, c.d);
  k_cell_scan<<<kp.R, 1024, 0, s>>>(kp, c.d);
  k_cell_scatter<<<ga, 128, 0, s>>>(kp, c.d);
  k_cell_sort<<<dim3((kp.ncell + 3) / 4, kp.R), 128, 0, s>>>(kp, c.d);
  k_permute<<<ga, 128, 0, s>>>(kp, c.d);
  k_copy_back<<<ga, 128, 0, s>>>(kp, c.d);
  return 6;
}

int launch_build_list(Ctx &c, cudaStream_t s) {
  if (c.kp.pair_mode == 1) {
    const size_t n = (size_t)c.kp.R * c.kp.nsc;
    cudaMemsetAsync(c.d.sc_ni, 0, sizeof(int) * n, s);
    cudaMemsetAsync(c.d.cl_n, 0, sizeof(int) * n, s);
    k_build_cluster<<<dim3(c.kp.nc[0] * c.kp.nc[1], c.kp.R), 32 * kClWarps, 0, s>>>(c.kp, c.d);
    if (c.kp.nlam) k_build_lam_list<<<dim3(c.kp.nlam, c.kp.R), 32, 0, s>>>(c.kp, c.d);
    return c.kp.nlam ? 2 : 1;
  }
  static const bool by_cell = getenv("CPH_BUILD") && getenv("CPH_BUILD")[0] == 'c';   // A/B: one warp per cell
  if (by_cell) k_build_list<<<dim3(c.kp.ncell, c.kp.R), 32, 0, s>>>(c.kp, c.d);
  else {
    const int ncol = c.kp.nc[0] * c.kp.nc[1];
    static const int force = getenv("CPH_COL_WARPS") ? atoi(getenv("CPH_COL_WARPS")) : 0;
    const bool small = force ? force == 4 : (double)c.kp.N / ncol <= 160.0;
    if (small) k_build_list_col<4><<<dim3(ncol, c.kp.R), 32 * 4, 0, s>>>(c.kp, c.d);
    else k_build_list_col<8><<<dim3(ncol, c.kp.R), 32 * 8, 0, s>>>(c.kp, c.d);
  }
  return 1;
}

int launch_rebuild(Ctx &c, cudaStream_t s) { return launch_sort(c, s) + launch_build_list(c, s); }

}  // namespace cph
