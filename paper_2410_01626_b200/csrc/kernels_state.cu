// Replica state blobs (cph_get_state / cph_set_state and the _all variants) on the device.
//
// Blob of one replica: int64 header (magic, N, C, step) | positions [3N] f32 | velocities [3N]
// f32 (original atom order) | lambda [C] f64 | lambda velocities [C] f64.  Packing and
// unpacking run as kernels (slot <-> original order through meta), so a whole batch moves
// host <-> device in one copy.
#include "cph_device.cuh"

namespace cph {

constexpr long long kStateMagic = 0x3148504331ll;

__global__ void k_pack_state(KParams kp, DevBufs d, char *dst, long long one, int r0, long long step) {
  const int r = r0 + blockIdx.y, s = blockIdx.x * blockDim.x + threadIdx.x;
  char *b = dst + (size_t)blockIdx.y * one;
  float *pos = reinterpret_cast<float *>(b + 32);
  float *vel = pos + 3 * (size_t)kp.N;
  double *lam = reinterpret_cast<double *>(vel + 3 * (size_t)kp.N);
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      long long *h = reinterpret_cast<long long *>(b);
      h[0] = kStateMagic; h[1] = kp.N; h[2] = kp.C; h[3] = step;
    }
    for (int c = threadIdx.x; c < kp.C; c += blockDim.x) {
      lam[c] = d.lam[(size_t)r * kp.C + c];
      lam[kp.C + c] = d.lamv[(size_t)r * kp.C + c];
    }
  }
  if (s >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + s;
  const int o = d.meta[idx].x;
  const float4 x = d.xyzq[idx], v = d.vel[idx];
  pos[3 * o] = x.x; pos[3 * o + 1] = x.y; pos[3 * o + 2] = x.z;
  vel[3 * o] = v.x; vel[3 * o + 1] = v.y; vel[3 * o + 2] = v.z;
}

__global__ void k_check_state(KParams kp, DevBufs d, const char *src, long long one) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const char *b = src + (size_t)blockIdx.y * one;
  const float *pos = reinterpret_cast<const float *>(b + 32);
  const double *lam = reinterpret_cast<const double *>(pos + 6 * (size_t)kp.N);
  bool bad = false;
  for (int k = s; k < 6 * kp.N; k += gridDim.x * blockDim.x) bad |= !isfinite(pos[k]);
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < 2 * kp.C; c += blockDim.x) bad |= !isfinite(lam[c]);
  if (bad) d.flags[FLAG_BAD_STATE] = 1;
}

__global__ void k_unpack_state(KParams kp, DevBufs d, const char *src, long long one, int r0) {
  const int r = r0 + blockIdx.y, s = blockIdx.x * blockDim.x + threadIdx.x;
  const char *b = src + (size_t)blockIdx.y * one;
  const float *pos = reinterpret_cast<const float *>(b + 32);
  const float *vel = pos + 3 * (size_t)kp.N;
  const double *lam = reinterpret_cast<const double *>(vel + 3 * (size_t)kp.N);
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < kp.C; c += blockDim.x) {
      d.lam[(size_t)r * kp.C + c] = lam[c];
      d.lamv[(size_t)r * kp.C + c] = lam[kp.C + c];
    }
  if (s >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + s;
  const int o = d.meta[idx].x;
  float4 x = d.xyzq[idx], v = d.vel[idx];
  x.x = pos[3 * o]; x.y = pos[3 * o + 1]; x.z = pos[3 * o + 2];
  d.xyzq[idx] = x;
  if (v.w > 0.0f) {                                  // frozen atoms keep zero velocity
    v.x = vel[3 * o]; v.y = vel[3 * o + 1]; v.z = vel[3 * o + 2];
    d.vel[idx] = v;
  }
}

// FLAG_MOVED = 1 when an atom of replicas [r0, r0 + nr) is not where it was at the last
// rebuild (xyzq_alt keeps the rebuild's wrapped positions until the next one): minimum-image
// displacement above 1e-5 nm.  Otherwise the pair list built there is the list of this
// configuration and a restore needs no re-sort and no rebuild.
__global__ void k_list_moved(KParams kp, DevBufs d, int r0) {
  const int r = r0 + blockIdx.y, s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= kp.N) return;
  const size_t idx = (size_t)r * kp.Nst + s;
  const float4 x = d.xyzq[idx], b = d.xyzq_alt[idx];
  float dx = x.x - b.x, dy = x.y - b.y, dz = x.z - b.z;
  dx -= kp.L[0] * rintf(dx * kp.invL[0]);
  dy -= kp.L[1] * rintf(dy * kp.invL[1]);
  dz -= kp.L[2] * rintf(dz * kp.invL[2]);
  if (!(dx * dx + dy * dy + dz * dz <= 1e-10f)) d.flags[FLAG_MOVED] = 1;
}

int launch_list_moved(Ctx &c, cudaStream_t s, int r0, int nr) {
  k_list_moved<<<dim3((c.kp.N + 255) / 256, nr), 256, 0, s>>>(c.kp, c.d, r0);
  return 1;
}

int launch_pack_state(Ctx &c, cudaStream_t s, char *dst, long long one, int r0, int nr, long long step) {
  k_pack_state<<<dim3((c.kp.N + 255) / 256, nr), 256, 0, s>>>(c.kp, c.d, dst, one, r0, step);
  return 1;
}
int launch_check_state(Ctx &c, cudaStream_t s, const char *src, long long one, int nr) {
  k_check_state<<<dim3(64, nr), 256, 0, s>>>(c.kp, c.d, src, one);
  return 1;
}
int launch_unpack_state(Ctx &c, cudaStream_t s, const char *src, long long one, int r0, int nr) {
  k_unpack_state<<<dim3((c.kp.N + 255) / 256, nr), 256, 0, s>>>(c.kp, c.d, src, one, r0);
  return 1;
}

}  // namespace cph
