// Host runtime behind include/cph.h: validation, device memory, PFC, cuFFT plans, step
// scheduling (CUDA graph per nstlist block, nonbonded || PME on two streams), getters.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "cph_device.cuh"

using namespace cph;

// NVTX ranges (header-only nvtx3): one per API call and per kernel class of an eagerly
// enqueued step, so an nsys / ncu --nvtx timeline attributes every launch
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define CPH_NVTX(name) NvtxRange nvtx_range_(name)

struct SubCtx {
  Ctx c;
};

namespace {

thread_local std::string g_create_err;

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      c.err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
      return CPH_E_CUDA;                                                          \
    }                                                                             \
  } while (0)

#define CKF(call)                                                                 \
  do {                                                                            \
    cufftResult r_ = (call);                                                      \
    if (r_ != CUFFT_SUCCESS) {                                                    \
      c.err = std::string(#call) + ": cuFFT error " + std::to_string((int)r_);    \
      return CPH_E_CUDA;                                                          \
    }                                                                             \
  } while (0)

template <class T>
T *dalloc(Ctx &c, size_t count) {
  size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  void *p = nullptr;
  if (c.dev_alloc) p = c.dev_alloc(bytes, c.alloc_ctx);
  else if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
  if (p) {
    c.allocations.push_back(p);
    cudaMemset(p, 0, bytes);
  }
  return (T *)p;
}

void free_all(Ctx &c) {
  for (void *p : c.allocations) {
    if (c.dev_free) c.dev_free(p, c.alloc_ctx);
    else cudaFree(p);
  }
  c.allocations.clear();
}

bool smooth2357(int k) {
  if (k <= 0) return false;
  for (int f : {2, 3, 5, 7})
    while (k % f == 0) k /= f;
  return k == 1;
}

double erfc_beta(double rc, double rtol) {
  double lo = 0.0, hi = 50.0 / rc;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (std::erfc(mid * rc) > rtol) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

double bspline4_at(double t) {   // M4 at integer arguments 1, 2, 3
  if (t == 1.0 || t == 3.0) return 1.0 / 6.0;
  if (t == 2.0) return 4.0 / 6.0;
  return 0.0;
}

void bsp_moduli(int K, std::vector<float> &out) {
  for (int m = 0; m < K; ++m) {
    double re = 0.0, im = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double a = 2.0 * kPi * m * k / K;
      re += bspline4_at(k + 1.0) * std::cos(a);
      im += bspline4_at(k + 1.0) * std::sin(a);
    }
    out.push_back((float)(1.0 / (re * re + im * im)));
  }
}

bool finite_arr(const float *p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}
bool finite_arr(const double *p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// PFC of replica r (all groups, or the groups flagged in `only`), with the current DBO
// parameters of each coordinate: host arithmetic only, results in h_d1 / h_dG
static bool compute_pfc_at(const Ctx &c, double pH, const double *dw, double *d1, double *dG,
                           const std::vector<char> *only, std::string *err) {
  const KParams &kp = c.kp;
  for (int g = 0; g < kp.G; ++g) {
    const double *pk = &c.h_pKa[(size_t)g * 3];
    for (int k = 0; k < 3; ++k) dG[(size_t)g * 3 + k] = delta_g(pk[k], pH, kp.kT / kBoltz);
    if (only && !(*only)[g]) continue;
    const int c0 = c.h_cptr[g];
    const bool ok = c.h_group_kind[g] == 2
                        ? pfc_two_state(dw + 4 * c0, pk[0], pH, kp.kT / kBoltz, kp.wall_k, &d1[c0], err)
                        : pfc_three_state(dw + 4 * c0, dw + 4 * (c0 + 1), pk, pH, kp.kT / kBoltz, kp.wall_k, &d1[c0],
                                          &d1[c0 + 1], err);
    if (!ok) return false;
  }
  return true;
}

static bool compute_pfc(Ctx &c, int r, const std::vector<char> *only, std::string *err) {
  const KParams &kp = c.kp;
  return compute_pfc_at(c, c.h_pH[r], c.h_dw.data() + (size_t)r * kp.C * 4, c.h_d1.data() + (size_t)r * kp.C,
                        c.h_dG.data() + (size_t)r * kp.G * 3, only, err);
}

// run f(k) for k in [0, n) on host threads
template <class F>
static void parallel_for(size_t n, F f) {
  const size_t nt = std::max<size_t>(1, std::min<size_t>(n, std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  auto work = [&]() {
    for (size_t k; (k = next.fetch_add(1)) < n;) f(k);
  };
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto &t : th) t.join();
}

// PFC for a set of replicas (host threads, one replica per task), then one upload
cph_status run_pfc_many(Ctx &c, const std::vector<int> &reps, const std::vector<std::vector<char>> *only = nullptr) {
  if (reps.empty()) return CPH_OK;
  std::atomic<bool> failed{false};
  std::string ferr;
  std::mutex mu;
  parallel_for(reps.size(), [&](size_t k) {
    std::string e;
    if (!compute_pfc(c, reps[k], only ? &(*only)[reps[k]] : nullptr, &e)) {
      std::lock_guard<std::mutex> lk(mu);
      failed = true;
      ferr = e;
    }
  });
  if (failed) { c.err = ferr; return CPH_E_INVALID; }
  const KParams &kp = c.kp;
  if (kp.C) CK(cudaMemcpy(c.d.d1, c.h_d1.data(), sizeof(double) * c.h_d1.size(), cudaMemcpyHostToDevice));
  if (kp.G) CK(cudaMemcpy(c.d.g_dG, c.h_dG.data(), sizeof(double) * c.h_dG.size(), cudaMemcpyHostToDevice));
  return CPH_OK;
}

// pH ladder: PFC once per level (undisturbed wells), every replica takes its level's rows
cph_status run_pfc_levels(Ctx &c, const std::vector<int> &labels) {
  const KParams &kp = c.kp;
  const int P = kp.P;
  c.h_lvl_d1.assign((size_t)P * kp.C, 0.0);
  c.h_lvl_dG.assign((size_t)P * kp.G * 3, 0.0);
  std::vector<double> dw0((size_t)kp.C * 4);
  for (int k = 0; k < kp.C; ++k) {
    dw0[4 * k] = 0.0; dw0[4 * k + 1] = 1.0; dw0[4 * k + 2] = dw0[4 * k + 3] = kp.h_barrier;
  }
  std::atomic<bool> failed{false};
  parallel_for(P, [&](size_t p) {
    std::string e;
    if (!compute_pfc_at(c, c.h_levels[p], dw0.data(), c.h_lvl_d1.data() + p * kp.C, c.h_lvl_dG.data() + p * kp.G * 3,
                        nullptr, &e))
      failed = true;
  });
  if (failed) { c.err = "PFC failed on the pH ladder"; return CPH_E_INVALID; }
  for (int r = 0; r < kp.R; ++r) {
    std::copy_n(c.h_lvl_d1.begin() + (size_t)labels[r] * kp.C, kp.C, c.h_d1.begin() + (size_t)r * kp.C);
    std::copy_n(c.h_lvl_dG.begin() + (size_t)labels[r] * kp.G * 3, kp.G * 3, c.h_dG.begin() + (size_t)r * kp.G * 3);
  }
  if (kp.C) {
    CK(cudaMemcpy(c.d.lvl_d1, c.h_lvl_d1.data(), sizeof(double) * c.h_lvl_d1.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.d.d1, c.h_d1.data(), sizeof(double) * c.h_d1.size(), cudaMemcpyHostToDevice));
  }
  if (kp.G) {
    CK(cudaMemcpy(c.d.lvl_dG, c.h_lvl_dG.data(), sizeof(double) * c.h_lvl_dG.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c.d.g_dG, c.h_dG.data(), sizeof(double) * c.h_dG.size(), cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(c.d.remd_label, labels.data(), sizeof(int) * kp.R, cudaMemcpyHostToDevice));
  return CPH_OK;
}

cph_status run_pfc(Ctx &c, int r) { return run_pfc_many(c, std::vector<int>{r}); }

__global__ void k_set_end(long long *end, long long v) { *end = v; }

// ---- timeline diagnostic (CPH_TIMELINE=1): timing events captured into the step graph at
// stage boundaries; mean offsets from each step's start are printed at cph_destroy
__global__ void k_stamp(unsigned long long *p) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *p = t;
}
static void tl_mark(Ctx &c, cudaStream_t st, int tag) {
  Timeline *t = c.tl;
  if (!t || t->s >= Timeline::S) return;
  k_stamp<<<1, 1, 0, st>>>(t->stamps + t->s * Timeline::T + tag);
  t->used[t->s][tag] = true;
}
static void tl_collect(Ctx &c) {
  Timeline *t = c.tl;
  if (!t) return;
  unsigned long long h[Timeline::S][Timeline::T];
  cudaStreamSynchronize(c.stream);
  cudaMemcpy(h, t->stamps, sizeof(h), cudaMemcpyDeviceToHost);
  for (int s = 0; s < Timeline::S; ++s)
    for (int k = 1; k < Timeline::T; ++k)
      if (t->used[s][k] && t->used[s][0]) t->sum[s][k] += 1e-3 * (double)(long long)(h[s][k] - h[s][0]);
  t->n += 1;
}
static void tl_print(Ctx &c) {
  Timeline *t = c.tl;
  if (!t || !t->n) return;
  static const char *names[Timeline::T] = {"start", "integrate", "sort", "build", "spread", "r2c", "solve", "c2r",
                                           "pair", "gather", "lambda", "-"};
  for (int s = 0; s < c.kp.nstlist && s < Timeline::S; ++s) {
    fprintf(stderr, "[timeline] step %d:", s);
    for (int k = 1; k < Timeline::T; ++k)
      if (t->used[s][k]) fprintf(stderr, " %s %.1f", names[k], t->sum[s][k] / t->n);
    fprintf(stderr, " (us, %d blocks)\n", t->n);
  }
}

// the PME transforms (fp32, or fp64 on small grids: kp.fft64), on the plans' current stream
static cufftResult fft_forward(Ctx &c) {
  if (c.kp.fft64) return cufftExecD2Z(c.plan_r2c, c.d.grid64, (cufftDoubleComplex *)c.d.cgrid64);
  return cufftExecR2C(c.plan_r2c, c.d.grid, (cufftComplex *)c.d.cgrid);
}
static cufftResult fft_backward(Ctx &c) {
  if (c.kp.fft64) return cufftExecZ2D(c.plan_c2r, (cufftDoubleComplex *)c.d.cgrid64, c.d.grid64);
  return cufftExecC2R(c.plan_c2r, (cufftComplex *)c.d.cgrid, c.d.grid);
}

// one full step (n -> n+1) on the context streams; returns kernels launched
int enqueue_step(Ctx &c, bool rebuild, bool two_streams) {
  CPH_NVTX(rebuild ? "cph step (rebuild)" : "cph step");
  int k = 0;
  cudaStream_t s = c.stream;
  tl_mark(c, s, 0);
  k += launch_integrate(c, s, 1);
  tl_mark(c, s, 1);
  static const bool serial_build = getenv("CPH_SERIAL_BUILD") != nullptr;   // A/B diagnostic
  if (rebuild) k += serial_build ? launch_rebuild(c, s) : launch_sort(c, s);
  if (rebuild) tl_mark(c, s, 2);
  cudaStream_t sp = s;
  if (two_streams) {
    cudaEventRecord(c.ev_fork, s);
    cudaStreamWaitEvent(c.stream_pme, c.ev_fork, 0);
    sp = c.stream_pme;
  }
  // the PME chain needs only the sorted atoms: it overlaps the list build
  if (rebuild && !serial_build) k += launch_build_list(c, s);
  if (rebuild) tl_mark(c, s, 3);
  cufftSetStream(c.plan_r2c, sp);
  cufftSetStream(c.plan_c2r, sp);
  k += launch_spread(c, sp);
  tl_mark(c, sp, 4);
  fft_forward(c);
  tl_mark(c, sp, 5);
  k += launch_solve(c, sp, 1);
  tl_mark(c, sp, 6);
  fft_backward(c);
  k += launch_grid_to32(c, sp);
  tl_mark(c, sp, 7);
  k += launch_hi_recip(c, sp);
  // the lambda kernel reads phi_rec of its atoms straight from the grid: it waits for the
  // back transform only, and the all-atom force gather runs beside it (joined below, before
  // anything that reads f_rec)
  if (two_streams) cudaEventRecord(c.ev_join, c.stream_pme);
  else k += launch_gather(c, s);
  static const bool lam_low = getenv("CPH_LAMBDA_LOWPRIO") != nullptr;   // A/B: round-1 placement
  if (two_streams && c.prio && !lam_low) {
    // the pair kernel on a high-priority stream: the PME chain (low priority) fills the SMs
    // the pair kernel leaves free instead of displacing its CTAs.  The lambda kernel (one CTA
    // per replica, the end of the step's critical path) follows on the same high-priority
    // stream once the back transform is done, so its CTAs are not queued behind the
    // all-atom gather's thousands of CTAs on the PME stream.
    cudaEventRecord(c.ev_fork2, s);
    cudaStreamWaitEvent(c.stream_nb, c.ev_fork2, 0);
    k += launch_nonbonded(c, c.stream_nb, 1);
    tl_mark(c, c.stream_nb, 8);
    k += launch_gather(c, c.stream_pme);
    tl_mark(c, c.stream_pme, 9);
    cudaEventRecord(c.ev_gather, c.stream_pme);
    cudaStreamWaitEvent(c.stream_nb, c.ev_join, 0);
    k += launch_hi_finish(c, c.stream_nb, 1);
    k += launch_lambda_reduce(c, c.stream_nb, 1);
    tl_mark(c, c.stream_nb, 10);
    cudaEventRecord(c.ev_join2, c.stream_nb);
    cudaStreamWaitEvent(s, c.ev_join2, 0);
    cudaStreamWaitEvent(s, c.ev_gather, 0);
    return k;
  }
  if (two_streams && c.prio) {
    cudaEventRecord(c.ev_fork2, s);
    cudaStreamWaitEvent(c.stream_nb, c.ev_fork2, 0);
    k += launch_nonbonded(c, c.stream_nb, 1);
    tl_mark(c, c.stream_nb, 8);
    cudaEventRecord(c.ev_join2, c.stream_nb);
    cudaStreamWaitEvent(s, c.ev_join2, 0);
  } else {
    k += launch_nonbonded(c, s, 1);
    tl_mark(c, s, 8);
  }
  if (two_streams) {
    cudaStreamWaitEvent(s, c.ev_join, 0);
    k += launch_gather(c, c.stream_pme);
    tl_mark(c, c.stream_pme, 9);
    cudaEventRecord(c.ev_gather, c.stream_pme);
  }
  k += launch_hi_finish(c, s, 1);
  k += launch_lambda_reduce(c, s, 1);
  tl_mark(c, s, 10);
  if (two_streams) cudaStreamWaitEvent(s, c.ev_gather, 0);
  return k;
}

// evaluation at the current state without integration (create / set_state)
// Forces, potentials and energies at the current state.  rebuild = false when the pair list of
// the last rebuild is the list of the current positions (they have not moved since, or the
// nstlist schedule covers them: a mid-run re-evaluation after a bias change).
cph_status evaluate_here(Ctx &c, bool rebuild) {
  CPH_NVTX("evaluate_here");
  cudaStream_t s = c.stream;
  k_set_end<<<1, 1, 0, s>>>(c.d.end_step, c.host_step);
  CK(cudaMemsetAsync(c.d.erec + (size_t)(c.host_step & 1) * c.kp.R * kNE, 0, sizeof(double) * c.kp.R * kNE, s));
  CK(cudaMemsetAsync(c.d.bussi_k, 0, sizeof(double) * 2 * c.kp.R, s));
  int k = 1;
  k += launch_set_charges(c, s);
  if (rebuild) k += launch_rebuild(c, s);
  // the PME chain on its own stream beside the pair kernel, joined before the lambda kernel
  // (as in a step; CPH_ONE_STREAM serialises both, a diagnostic)
  static const bool one = getenv("CPH_ONE_STREAM") != nullptr;
  cudaStream_t sp = s;
  if (!one) {
    CK(cudaEventRecord(c.ev_fork, s));
    CK(cudaStreamWaitEvent(c.stream_pme, c.ev_fork, 0));
    sp = c.stream_pme;
  }
  cufftSetStream(c.plan_r2c, sp);
  cufftSetStream(c.plan_c2r, sp);
  k += launch_spread(c, sp);
  CKF(fft_forward(c));
  k += launch_solve(c, sp, 0);
  CKF(fft_backward(c));
  k += launch_grid_to32(c, sp);
  k += launch_gather(c, sp);
  k += launch_hi_recip(c, sp);
  if (!one) CK(cudaEventRecord(c.ev_join, sp));
  k += launch_nonbonded(c, s, 0);
  if (!one) CK(cudaStreamWaitEvent(s, c.ev_join, 0));
  k += launch_hi_finish(c, s, 0);
  k += launch_lambda_reduce(c, s, 0);
  k += launch_close(c, s, 0);
  c.launches += k;
  CK(cudaGetLastError());
  return CPH_OK;
}

cph_status check_flags(Ctx &c) {
  int f[FLAG_COUNT];
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaMemcpy(f, c.d.flags, sizeof(f), cudaMemcpyDeviceToHost));
  if (f[FLAG_DIVERGED]) {
    c.err = "lambda diverged (|lambda| > 10 or non-finite dV/dlambda)";
    return CPH_E_DIVERGED;
  }
  if (f[FLAG_REMD_BAD]) {
    c.err = "replica exchange: gathered labels do not form ladders (a level missing or held twice); no swap was made";
    return CPH_E_STATE;
  }
  if (f[FLAG_LIST_OVERFLOW]) {
    char buf[160];
    snprintf(buf, sizeof buf, "pair list overflow: %d neighbours > capacity %d; results since the last rebuild are invalid",
             f[FLAG_MAX_NNB], c.kp.cap);
    c.err = buf;
    c.cap_grow = (size_t)f[FLAG_MAX_NNB];
    if (f[FLAG_CL_OVERFLOW]) c.clcap_grow = (size_t)f[FLAG_CL_MAX];
    return CPH_E_STATE;
  }
  if (f[FLAG_CL_OVERFLOW]) {
    char buf[160];
    snprintf(buf, sizeof buf, "cluster pair list overflow: %d entries > capacity %d; results since the last rebuild are invalid",
             f[FLAG_CL_MAX], c.kp.clcap);
    c.err = buf;
    c.clcap_grow = (size_t)f[FLAG_CL_MAX];
    return CPH_E_STATE;
  }
  return CPH_OK;
}

cph_status capture_block(Ctx &c) {
  if (c.graph_block) return CPH_OK;
  cudaGraph_t g;
  if (getenv("CPH_TIMELINE") && !c.tl) {
    c.tl = new Timeline();
    CK(cudaMalloc(&c.tl->stamps, sizeof(unsigned long long) * Timeline::S * Timeline::T));
  }
  CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  int k = 0;
  const bool two = getenv("CPH_ONE_STREAM") == nullptr;   // diagnostic switch: serialise NB and PME
  for (int s = 0; s < c.kp.nstlist; ++s) {
    if (c.tl) c.tl->s = s;
    k += enqueue_step(c, s == c.kp.nstlist - 1, two);
  }
  if (c.tl) c.tl->s = Timeline::S;   // eager steps are not marked
  CK(cudaStreamEndCapture(c.stream, &g));
  CK(cudaGraphInstantiateWithFlags(&c.graph_block, g, c.prio ? cudaGraphInstantiateFlagUseNodePriority : 0));
  cudaGraphDestroy(g);
  c.graph_block_kernels = k;
  return CPH_OK;
}

// Every ladder (P consecutive global replicas) that lies entirely inside [first, first + R)
// must hold each level 0..P-1 exactly once (R29); partially held ladders are checked
// on the device at each exchange (k_remd_apply).
bool labels_form_ladders(const int *labels, int R, int first, int P) {
  for (int l0 = (first + P - 1) / P * P; l0 + P <= first + R; l0 += P) {
    std::vector<char> seen(P, 0);
    for (int g = l0; g < l0 + P; ++g) {
      const int lab = labels[g - first];
      if (lab < 0 || lab >= P || seen[lab]) return false;
      seen[lab] = 1;
    }
  }
  return true;
}

cph_status check_replica(Ctx &c, int r) {
  if (r < 0 || r >= c.kp.R) {
    c.err = "replica index out of range";
    return CPH_E_INVALID;
  }
  return CPH_OK;
}

}  // namespace


void cph_default_params(cph_params *p) {
  std::memset(p, 0, sizeof(*p));
  p->abi_version = CPH_ABI_VERSION;
  p->n_replicas = 1;
  p->dt = 0.002;
  p->temperature = 300.0;
  p->gamma_atom = 1.0;
  p->gamma_lambda = 1.0;
  p->lambda_mass = 60.0;
  p->rc = 1.0;
  p->rlist = 1.1;
  p->ewald_rtol = 1e-5;
  p->pme_grid[0] = p->pme_grid[1] = p->pme_grid[2] = 32;
  p->pme_order = 4;
  p->nstlist = 10;
  p->nstout = 250;
  p->nstenergy = 250;
  p->barrier = 6.0;
  p->wall_k = 1e6;
  p->frame_capacity = 1024;
  p->dbo_well = 0;
  p->dbo_barrier = 0;
  p->dbo_well_steps = 20000;       // 40 ps
  p->dbo_barrier_steps = 500000;   // 1 ns
  p->dbo_censor_steps = 5000;      // 10 ps
  p->dbo_well_near = 0.2;
  p->dbo_residency = 0.7;
  p->dbo_well_tol = 0.03;
  p->dbo_well_gain = 0.5;
  p->dbo_well_cap = 0.08;
  p->dbo_trans_lo = 0.2;
  p->dbo_trans_hi = 0.8;
  p->dbo_target = 0.25;
  p->dbo_target_tol = 0.05;
  p->dbo_barrier_step = 1.0;
  p->dbo_barrier_min = 1.0;
  p->dbo_barrier_max = 20.0;
  p->thermostat = 0;
  p->tau_atom = 0.1;
  p->tau_lambda = 1.0;
  p->n_ph_levels = 0;
  p->ph_levels = nullptr;
  p->remd_first = 0;
  p->remd_total = 0;
  p->hamiltonian = 0;
  p->deterministic = 0;
  p->sub_batches = 0;
  p->pair_list = 0;
}


static cph_status fail_create(SubCtx *ctx, cph_status st) {
  g_create_err = ctx->c.err;
  free_all(ctx->c);
  delete ctx;
  return st;
}

static cph_status sub_create(const cph_system *sys, const cph_params *prm, SubCtx **out) {
  CPH_NVTX("cph_create");
  if (!out) { g_create_err = "out is NULL"; return CPH_E_INVALID; }
  *out = nullptr;
  if (!sys || !prm) { g_create_err = "system/params is NULL"; return CPH_E_INVALID; }
  SubCtx *ctx = new SubCtx;
  Ctx &c = ctx->c;
  auto bad = [&](const char *m) { c.err = m; return fail_create(ctx, CPH_E_INVALID); };
  if (prm->abi_version != CPH_ABI_VERSION) return bad("abi_version mismatch");
  const int N = sys->n_atoms, R = prm->n_replicas, G = sys->n_groups, T = sys->n_types;
  if (N < 1 || N > kMaxAtoms) return bad("n_atoms must be in [1, 2^21]");
  if (R < 1) return bad("n_replicas must be >= 1");
  if (!sys->pos || !sys->mass || !sys->charge || !sys->type || !sys->c6 || !sys->c12)
    return bad("system arrays pos/mass/charge/type/c6/c12 are required");
  if (T < 1 || T > kMaxTypes) return bad("n_types must be in [1, 32]");
  if (!finite_arr(sys->pos, 3 * (size_t)N) || !finite_arr(sys->mass, N) || !finite_arr(sys->charge, N) ||
      (sys->vel && !finite_arr(sys->vel, 3 * (size_t)N)) || !finite_arr(sys->c6, (size_t)T * T) ||
      !finite_arr(sys->c12, (size_t)T * T) || !finite_arr(sys->box, 3))
    return bad("non-finite value in system");
  for (int i = 0; i < N; ++i) {
    if (sys->mass[i] < 0.0f) return bad("negative mass");
    if (sys->type[i] < 0 || sys->type[i] >= T) return bad("type out of range");
  }
  for (int d = 0; d < 3; ++d)
    if (!(sys->box[d] > 0.0)) return bad("box edges must be > 0");
  if (!(prm->rc > 0.0) || !(prm->rlist >= prm->rc)) return bad("need 0 < rc <= rlist");
  for (int d = 0; d < 3; ++d)
    if (!(prm->rlist < 0.5 * sys->box[d])) return bad("rlist must be < half of every box edge");
  if (!(prm->dt > 0.0) || !(prm->temperature > 0.0) || !(prm->lambda_mass > 0.0) || prm->gamma_atom < 0.0 ||
      prm->gamma_lambda < 0.0 || !(prm->ewald_rtol > 0.0 && prm->ewald_rtol < 1.0))
    return bad("invalid dynamics / Ewald parameter");
  if (prm->nstlist < 1 || prm->nstout < 1 || prm->nstenergy < 1 || prm->frame_capacity < 1)
    return bad("nstlist, nstout, nstenergy, frame_capacity must be >= 1");
  if (prm->mode != 0 && prm->mode != 1) return bad("mode must be 0 or 1");
  if (prm->thermostat != 0 && prm->thermostat != 1) return bad("thermostat must be 0 (Langevin) or 1 (Bussi)");
  if (prm->hamiltonian != 0 && prm->hamiltonian != 1) return bad("hamiltonian must be 0 or 1");
  if (prm->deterministic != 0 && prm->deterministic != 1) return bad("deterministic must be 0 or 1");
  if (prm->pair_list < 0 || prm->pair_list > 2) return bad("pair_list must be 0, 1 or 2");
  if (prm->deterministic && prm->pair_list == 2) return bad("deterministic = 1 needs the per-atom pair list (pair_list 0 or 1)");
  if (prm->thermostat == 1 && !(prm->tau_atom > 0.0 && prm->tau_lambda > 0.0))
    return bad("Bussi coupling times must be > 0");
  std::vector<int> labels0;
  if (prm->n_ph_levels != 0) {
    const int P = prm->n_ph_levels;
    if (P < 2 || !prm->ph_levels || !finite_arr(prm->ph_levels, P)) return bad("replica exchange needs n_ph_levels >= 2 finite ph_levels");
    for (int p = 1; p < P; ++p)
      if (!(prm->ph_levels[p] > prm->ph_levels[p - 1])) return bad("ph_levels must be strictly ascending");
    if (prm->mode != 0 || prm->dbo_well || prm->dbo_barrier) {
      c.err = "pH replica exchange is not combinable with DBO or fixed-lambda mode";
      return fail_create(ctx, CPH_E_UNSUPPORTED);
    }
    const int total = prm->remd_total ? prm->remd_total : R;
    if (total % P || prm->remd_first < 0 || prm->remd_first + R > total)
      return bad("remd_total must be a multiple of n_ph_levels and hold [remd_first, remd_first + R)");
    if (!prm->pH) return bad("pH array is required");
    for (int r = 0; r < R; ++r) {
      int lab = -1;
      for (int p = 0; p < P; ++p)
        if (std::fabs(prm->pH[r] - prm->ph_levels[p]) <= 1e-9 * std::max(1.0, std::fabs(prm->ph_levels[p]))) lab = p;
      if (lab < 0) return bad("every replica pH must be one of ph_levels");
      labels0.push_back(lab);
    }
    c.h_levels.assign(prm->ph_levels, prm->ph_levels + P);
    if (!labels_form_ladders(labels0.data(), R, prm->remd_first, P))
      return bad("each pH ladder held by this context must carry every level exactly once");
  }
  if (prm->dbo_well || prm->dbo_barrier) {
    if ((prm->dbo_well && (prm->dbo_well_steps < 1 || prm->dbo_well_steps % prm->nstlist)) ||
        (prm->dbo_barrier && (prm->dbo_barrier_steps < 1 || prm->dbo_barrier_steps % prm->nstlist)) ||
        prm->dbo_censor_steps < 0)
      return bad("DBO block lengths must be positive multiples of nstlist, censor window >= 0");
    if (!(prm->dbo_well_near > 0.0 && prm->dbo_well_near < 0.5) || !(prm->dbo_residency >= 0.0) ||
        !(prm->dbo_well_tol >= 0.0) || !(prm->dbo_well_gain >= 0.0) ||
        !(prm->dbo_well_cap >= 0.0 && prm->dbo_well_cap <= 0.2) ||
        !(prm->dbo_trans_lo < prm->dbo_trans_hi) || !(prm->dbo_barrier_step >= 0.0) ||
        !(prm->dbo_barrier_min > 0.0 && prm->dbo_barrier_min <= prm->dbo_barrier_max && prm->dbo_barrier_max <= 100.0))
      return bad("invalid DBO rule constant");
  }
  if (!prm->pH || !prm->replica_seed) return bad("pH and replica_seed arrays are required");
  if (!finite_arr(prm->pH, R)) return bad("non-finite pH");
  if (prm->pme_order != 4) { c.err = "only pme_order 4 is implemented"; return fail_create(ctx, CPH_E_UNSUPPORTED); }
  for (int d = 0; d < 3; ++d)
    if (prm->pme_grid[d] < 8 || prm->pme_grid[d] % 2 || !smooth2357(prm->pme_grid[d])) {
      c.err = "PME grid dimensions must be even, >= 8 and 2,3,5,7-smooth";
      return fail_create(ctx, CPH_E_UNSUPPORTED);
    }
  // exclusions
  std::vector<std::vector<int>> ex(N);
  if (sys->n_excl < 0 || (sys->n_excl > 0 && !sys->excl)) return bad("bad exclusion list");
  for (int e = 0; e < sys->n_excl; ++e) {
    const int a = sys->excl[2 * e], b = sys->excl[2 * e + 1];
    if (a < 0 || b < 0 || a >= N || b >= N || a == b) return bad("exclusion index out of range or i == j");
    ex[a].push_back(b);
    ex[b].push_back(a);
  }
  c.h_excl_ptr.assign(N + 1, 0);
  for (int i = 0; i < N; ++i) {
    std::sort(ex[i].begin(), ex[i].end());
    ex[i].erase(std::unique(ex[i].begin(), ex[i].end()), ex[i].end());
    c.h_excl_ptr[i + 1] = c.h_excl_ptr[i] + (int)ex[i].size();
    c.h_excl_idx.insert(c.h_excl_idx.end(), ex[i].begin(), ex[i].end());
  }
  // lambda groups
  if (G < 0) return bad("n_groups < 0");
  int nlam = 0;
  std::vector<int> lslot(N, -1);
  c.h_cptr.assign(G + 1, 0);
  if (G > 0) {
    if (!sys->group_kind || !sys->group_ptr || !sys->group_atoms || !sys->state_q || !sys->pKa || !sys->vmm)
      return bad("group arrays are required when n_groups > 0");
    if (sys->group_ptr[0] != 0) return bad("group_ptr[0] must be 0");
    for (int g = 0; g < G; ++g) {
      const int k = sys->group_kind[g];
      if (k != 2 && k != 3) return bad("group_kind must be 2 or 3");
      if (sys->group_ptr[g + 1] <= sys->group_ptr[g]) return bad("empty lambda-group");
      c.h_cptr[g + 1] = c.h_cptr[g] + (k == 2 ? 1 : 2);
    }
    nlam = sys->group_ptr[G];
    if (!finite_arr(sys->state_q, 4 * (size_t)nlam) || !finite_arr(sys->pKa, 3 * (size_t)G) ||
        !finite_arr(sys->vmm, 36 * (size_t)G))
      return bad("non-finite group parameter");
    for (int g = 0; g < G; ++g) {
      double tot[4] = {0, 0, 0, 0};
      for (int k = sys->group_ptr[g]; k < sys->group_ptr[g + 1]; ++k) {
        const int a = sys->group_atoms[k];
        if (a < 0 || a >= N) return bad("group atom out of range");
        if (lslot[a] >= 0) return bad("atom belongs to more than one lambda-group");
        lslot[a] = k;
        const double *q = sys->state_q + 4 * (size_t)k;
        for (int s = 0; s < 4; ++s) tot[s] += q[s];
        if (sys->group_kind[g] == 2 && (std::fabs(q[0] - q[1]) > 1e-12 || std::fabs(q[2] - q[3]) > 1e-12))
          return bad("2-state group requires q^A == q^B and q^C == q^D");
      }
      for (int s = 1; s < 4; ++s)
        if (std::fabs(tot[s] - tot[0]) > 1e-9)
          return bad("lambda-group total charge varies between forms (site + buffer must be constant, PAPER.md:817)");
    }
    c.h_group_kind.assign(sys->group_kind, sys->group_kind + G);
    c.h_group_ptr.assign(sys->group_ptr, sys->group_ptr + G + 1);
    c.h_group_atoms.assign(sys->group_atoms, sys->group_atoms + nlam);
    c.h_state_q.assign(sys->state_q, sys->state_q + 4 * (size_t)nlam);
    c.h_pKa.assign(sys->pKa, sys->pKa + 3 * (size_t)G);
  }
  const int C = c.h_cptr[G];
  if (prm->hamiltonian)
    for (int g = 0; g < G; ++g)
      if (c.h_group_ptr[g + 1] - c.h_group_ptr[g] > 32) {
        c.err = "Hamiltonian interpolation supports lambda-groups of at most 32 atoms";
        return fail_create(ctx, CPH_E_UNSUPPORTED);
      }
  if (nlam > 12000) { c.err = "more than 12000 lambda atoms per replica"; return fail_create(ctx, CPH_E_UNSUPPORTED); }
  if (prm->lambda0 && !finite_arr(prm->lambda0, (size_t)R * C)) return bad("non-finite lambda0");

  // ---- kernel parameters ------------------------------------------------------------
  KParams &kp = c.kp;
  kp.R = R; kp.N = N; kp.Nst = (N + 31) / 32 * 32;
  double V = 1.0;
  for (int d = 0; d < 3; ++d) {
    kp.Ld[d] = sys->box[d];
    kp.L[d] = (float)sys->box[d];
    kp.invL[d] = 1.0f / kp.L[d];
    V *= sys->box[d];
  }
  kp.V = (float)V;
  {
    const float rcf = (float)prm->rc, rlf = (float)prm->rlist;
    kp.rc2 = rcf * rcf;
    kp.rlist2 = rlf * rlf;
  }
  kp.beta_d = erfc_beta(prm->rc, prm->ewald_rtol);
  kp.beta = (float)kp.beta_d;
  kp.beta_p = kp.beta * kErfcP;
  kp.two_beta_sqrtpi = (float)(2.0 * kp.beta_d / std::sqrt(kPi));
  kp.fcoul = (float)kFCoul;
  kp.T = T;
  kp.ncell = 1;
  for (int d = 0; d < 3; ++d) {
    int nc = (int)std::floor(sys->box[d] / (0.5 * prm->rlist * (1.0 + 1e-4)));
    if (nc < 1) nc = 1;
    kp.nc[d] = nc;
    if (nc >= 5) { kp.ns[d] = 5; kp.so[d] = -2; }
    else { kp.ns[d] = nc; kp.so[d] = 0; }
    kp.ncell *= nc;
  }
  kp.nb_packed = getenv("CPH_NB_PACKED") ? atoi(getenv("CPH_NB_PACKED")) : 1;
  kp.det = prm->deterministic;
  // pair-list layout (cph_params.pair_list): automatic = the per-atom full list, which is the
  // faster one on B200 (the cluster-pair kernel evaluates 757 pair slots per atom
  // against 578 list entries and issues 1.7x the instructions); CPH_PAIR=atom|cluster overrides
  // the automatic choice for A/B runs.  Deterministic mode needs the per-atom list (the cluster
  // kernel's j-side float4 reductions are order-dependent).
  kp.pair_mode = prm->pair_list == 2 ? 1 : 0;
  if (prm->pair_list == 0 && getenv("CPH_PAIR")) kp.pair_mode = getenv("CPH_PAIR")[0] == 'c' ? 1 : 0;
  if (kp.det) kp.pair_mode = 0;
  {
    const double expect = (double)N / V * 4.0 / 3.0 * kPi * std::pow(prm->rlist, 3);
    kp.cap = (int)std::ceil(1.6 * expect + 64.0);
    kp.cap = (kp.cap + 7) / 8 * 8;
    // cluster mode: super-cluster ids and entry capacity.  Entries of a super-cluster ~ the
    // j-clusters (4 atoms) within r_list of its region (one cell column wide, 32 atoms tall),
    // half of them (each pair once): rho V / 8 with V the region dilated by r_list + 0.15 nm
    // (the j-cluster extent), with a 2.5x margin (the mean is ~ 240 at density 100 nm^-3, dense solute regions reach ~1.8x)
    int ncol = 1;
    for (int d = 0; d < 2; ++d) ncol *= std::max(1, (int)std::floor(sys->box[d] / (0.5 * prm->rlist * (1.0 + 1e-4))));
    kp.nsc = kp.Nst / kClSuper + ncol + 1;
    const double rho = (double)N / V;
    const double ca = std::sqrt(sys->box[0] * sys->box[1] / ncol), cz = kClSuper / (rho * ca * ca);
    const double Rr = prm->rlist + 0.15;
    const double Vm = ca * ca * cz + 2.0 * (ca * ca + 2.0 * ca * cz) * Rr + kPi * (2.0 * ca + cz) * Rr * Rr +
                      4.0 / 3.0 * kPi * Rr * Rr * Rr;
    kp.clcap = (int)std::ceil(2.5 * rho * Vm / 8.0 + 128.0);
  }
  for (int d = 0; d < 3; ++d) kp.K[d] = prm->pme_grid[d];
  kp.K3 = kp.K[0] * kp.K[1] * kp.K[2];
  kp.fft64 = kp.K3 <= 32768;   // small grids: fp64 PME grid / transforms (kernels_pme.cu k_spread64)
  if (getenv("CPH_FFT64")) kp.fft64 = atoi(getenv("CPH_FFT64"));
  kp.Kzc = kp.K[2] / 2 + 1;
  kp.Kc = kp.K[0] * kp.K[1] * kp.Kzc;
  kp.dtd = prm->dt;
  kp.dt = (float)prm->dt;
  kp.kT = kBoltz * prm->temperature;
  kp.kT_f = (float)kp.kT;
  {
    const double c1 = std::exp(-prm->gamma_atom * prm->dt);
    kp.c1_atom = (float)c1;
    kp.c2_atom_kT = (float)((1.0 - c1 * c1) * kp.kT);
    const double cl = std::exp(-prm->gamma_lambda * prm->dt);
    kp.c1_lam = cl;
    kp.sd_lam = std::sqrt((1.0 - cl * cl) * kp.kT / prm->lambda_mass);
    kp.m_lam = prm->lambda_mass;
  }
  kp.nstout = prm->nstout;
  kp.nstenergy = prm->nstenergy;
  kp.nstlist = prm->nstlist;
  kp.mode = prm->mode;
  kp.G = G; kp.C = C; kp.nlam = nlam;
  kp.h_barrier = prm->barrier;
  kp.wall_k = prm->wall_k;
  kp.fcap = prm->frame_capacity;
  {
    DboConfig &b = c.dbo;
    const bool on = prm->mode == 0 && (prm->dbo_well || prm->dbo_barrier);
    b.well = on && prm->dbo_well;
    b.barrier = on && prm->dbo_barrier;
    b.well_steps = prm->dbo_well_steps; b.barrier_steps = prm->dbo_barrier_steps;
    b.censor_steps = prm->dbo_censor_steps;
    b.near = prm->dbo_well_near; b.residency = prm->dbo_residency; b.tol = prm->dbo_well_tol;
    b.gain = prm->dbo_well_gain; b.cap = prm->dbo_well_cap;
    b.trans_lo = prm->dbo_trans_lo; b.trans_hi = prm->dbo_trans_hi;
    b.target = prm->dbo_target; b.target_tol = prm->dbo_target_tol;
    b.bstep = prm->dbo_barrier_step; b.bmin = prm->dbo_barrier_min; b.bmax = prm->dbo_barrier_max;
    kp.dbo_on = on ? 1 : 0;
    kp.dbo_near = b.near; kp.dbo_trans_lo = b.trans_lo; kp.dbo_trans_hi = b.trans_hi;
  }
  kp.P = prm->n_ph_levels;
  kp.remd_total = kp.P ? (prm->remd_total ? prm->remd_total : R) : 0;
  kp.remd_first = kp.P ? prm->remd_first : 0;
  kp.hi = prm->hamiltonian == 1 && G > 0;
  std::vector<int4> hi_m;
  std::vector<float> hi_w;
  if (kp.hi) {
    // half-space m with exp(-pi^2 m^2/beta^2) >= 1e-8 (R31), 2 g(m) weights
    const double mmax2 = -std::log(1e-8) * kp.beta_d * kp.beta_d / (kPi * kPi);
    for (int e = 0; e < 3; ++e) kp.hi_kmax[e] = (int)std::floor(std::sqrt(mmax2) * sys->box[e]);
    for (int nz = 0; nz <= kp.hi_kmax[2]; ++nz)
      for (int ny = -kp.hi_kmax[1]; ny <= kp.hi_kmax[1]; ++ny)
        for (int nx = -kp.hi_kmax[0]; nx <= kp.hi_kmax[0]; ++nx) {
          if (nz == 0 && (ny < 0 || (ny == 0 && nx <= 0))) continue;
          const double mx = nx / sys->box[0], my = ny / sys->box[1], mz = nz / sys->box[2];
          const double m2 = mx * mx + my * my + mz * mz;
          if (m2 > mmax2) continue;
          hi_m.push_back(make_int4(nx, ny, nz, 0));
          hi_w.push_back((float)(2.0 * std::exp(-kPi * kPi * m2 / (kp.beta_d * kp.beta_d)) / (kPi * V * m2)));
        }
    kp.hi_nm = (int)hi_m.size();
    const int want = (2 * 148 + G * R - 1) / (G * R);
    kp.hi_nsplit = std::max(1, std::min((kp.hi_nm + 255) / 256, want));
  }
  kp.bussi = prm->thermostat == 1;
  {
    int mobile = 0;
    for (int i = 0; i < N; ++i) mobile += sys->mass[i] > 0.0f;
    kp.nf_atom = 3.0 * mobile;
    kp.cb_atom = kp.bussi ? std::exp(-prm->dt / prm->tau_atom) : 1.0;
    kp.cb_lam = kp.bussi ? std::exp(-prm->dt / prm->tau_lambda) : 1.0;
  }
  kp.Q_fixed = 0.0; kp.Q2_fixed = 0.0;
  for (int i = 0; i < N; ++i)
    if (lslot[i] < 0) { kp.Q_fixed += sys->charge[i]; kp.Q2_fixed += (double)sys->charge[i] * sys->charge[i]; }

  // ---- device ------------------------------------------------------------------------
  c.device = prm->device;
  if (cudaSetDevice(prm->device) != cudaSuccess) { c.err = "cudaSetDevice failed"; return fail_create(ctx, CPH_E_CUDA); }
  c.dev_alloc = prm->dev_alloc;
  c.dev_free = prm->dev_free;
  c.alloc_ctx = prm->alloc_ctx;
  if (prm->cuda_stream) c.stream = (cudaStream_t)prm->cuda_stream;
  else {
    if (cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess) {
      c.err = "stream creation failed";
      return fail_create(ctx, CPH_E_CUDA);
    }
    c.own_stream = true;
  }
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  c.prio = getenv("CPH_NO_PRIO") == nullptr && prio_hi != prio_lo;
  // A/B diagnostic: CPH_PRIO_SWAP=1 puts the PME chain on the high-priority stream instead
  static const bool swap = getenv("CPH_PRIO_SWAP") != nullptr;
  if (swap) std::swap(prio_lo, prio_hi);
  if (cudaStreamCreateWithPriority(&c.stream_nb, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_join2, cudaEventDisableTiming) != cudaSuccess) {
    c.err = "stream/event creation failed";
    return fail_create(ctx, CPH_E_CUDA);
  }
  if (cudaStreamCreateWithPriority(&c.stream_pme, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c.ev_gather, cudaEventDisableTiming) != cudaSuccess) {
    c.err = "stream/event creation failed";
    return fail_create(ctx, CPH_E_CUDA);
  }
  DevBufs &d = c.d;
  const size_t RN = (size_t)R * kp.Nst;
  d.xyzq = dalloc<float4>(c, RN); d.xyzq_alt = dalloc<float4>(c, RN);
  d.vel = dalloc<float4>(c, RN); d.vel_alt = dalloc<float4>(c, RN);
  d.meta = dalloc<int2>(c, RN); d.meta_alt = dalloc<int2>(c, RN);
  d.f_nb = dalloc<float4>(c, RN); d.f_rec = dalloc<float4>(c, RN);
  d.iperm = dalloc<int>(c, (size_t)R * N);
  d.cell_of = dalloc<int>(c, RN); d.cell_rank = dalloc<int>(c, RN);
  d.cell_count = dalloc<int>(c, (size_t)R * kp.ncell);
  d.cell_start = dalloc<int>(c, (size_t)R * (kp.ncell + 1));
  d.perm_tmp = dalloc<int>(c, RN);
  if (kp.pair_mode == 0) {
    d.nbl = dalloc<uint32_t>(c, RN * kp.cap);
    d.nnb = dalloc<int>(c, RN);
  } else {
    const size_t ns = (size_t)R * kp.nsc;
    d.cl_j = dalloc<uint32_t>(c, ns * kp.clcap);
    d.cl_m = dalloc<uint4>(c, ns * kp.clcap);
    d.cl_n = dalloc<int>(c, ns);
    d.sc_first = dalloc<int>(c, ns);
    d.sc_ni = dalloc<int>(c, ns);
    d.lam_nbl = dalloc<uint32_t>(c, std::max<size_t>(1, (size_t)R * nlam * kp.cap));
    d.lam_n = dalloc<int>(c, std::max<size_t>(1, (size_t)R * nlam));
    if (!d.cl_j || !d.cl_m || !d.cl_n || !d.sc_first || !d.sc_ni || !d.lam_nbl || !d.lam_n) {
      c.err = "device allocation failed";
      return fail_create(ctx, CPH_E_OOM);
    }
  }
  d.excl_ptr = dalloc<int>(c, N + 1);
  d.excl_idx = dalloc<int>(c, c.h_excl_idx.size());
  d.ljtab = dalloc<float2>(c, (size_t)T * T);
  d.phi64_nb = dalloc<double>(c, (size_t)R * nlam);
  d.phi_lam = dalloc<double>(c, (size_t)R * nlam);
  d.grid = dalloc<float>(c, (size_t)R * kp.K3);
  d.cgrid = dalloc<float2>(c, (size_t)R * kp.Kc);
  d.bsp = dalloc<float>(c, kp.K[0] + kp.K[1] + kp.K[2]);
  d.ginf = dalloc<float>(c, kp.Kc);
  if (kp.fft64) {
    d.grid64 = dalloc<double>(c, (size_t)R * kp.K3);
    d.cgrid64 = dalloc<double2>(c, (size_t)R * kp.Kc);
    d.ginf64 = dalloc<double>(c, kp.Kc);
    if (!d.grid64 || !d.cgrid64 || !d.ginf64) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
  }
  if (kp.det) {
    d.grid_fx = dalloc<unsigned long long>(c, (size_t)R * kp.K3);
    if (!d.grid_fx) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
  }
  d.g_kind = dalloc<int>(c, G); d.g_ptr = dalloc<int>(c, G + 1);
  d.g_atoms = dalloc<int>(c, nlam); d.g_cptr = dalloc<int>(c, G + 1);
  d.g_q = dalloc<double>(c, 4 * (size_t)nlam);
  d.k_group = dalloc<int>(c, nlam);
  d.vmm = dalloc<double>(c, 36 * (size_t)G);
  d.g_dG = dalloc<double>(c, (size_t)R * G * 3);
  d.d1 = dalloc<double>(c, (size_t)R * C);
  d.lam = dalloc<double>(c, (size_t)R * C); d.lamv = dalloc<double>(c, (size_t)R * C);
  d.qlam = dalloc<double>(c, (size_t)R * nlam);
  d.dvdl_coul = dalloc<double>(c, (size_t)R * C); d.dvdl_bias = dalloc<double>(c, (size_t)R * C);
  d.ti_sum = dalloc<double>(c, (size_t)R * C);
  d.ti_n = dalloc<long long>(c, 1);
  d.erec = dalloc<double>(c, 2 * (size_t)R * kNE);
  d.frames = dalloc<float>(c, (size_t)R * kp.fcap * C);
  d.frame_total = dalloc<long long>(c, R);
  d.step = dalloc<long long>(c, 1); d.end_step = dalloc<long long>(c, 1);
  d.done_counter = dalloc<int>(c, 1);
  d.flags = dalloc<int>(c, FLAG_COUNT);
  d.seed = dalloc<uint64_t>(c, R);
  d.dw = dalloc<double>(c, (size_t)R * C * 4);
  d.dbo_well = dalloc<double>(c, (size_t)R * C * 5);
  d.dbo_bar = dalloc<double>(c, (size_t)R * C * 4);
  d.c_group = dalloc<int>(c, C);
  d.c_lp = dalloc<int>(c, C);
  d.cens = dalloc<long long>(c, (size_t)R * G * 2);
  d.frame_cens = dalloc<unsigned char>(c, (size_t)R * kp.fcap * C);
  d.frame_step = dalloc<long long>(c, (size_t)R * kp.fcap);
  d.bussi_k = dalloc<double>(c, 2 * (size_t)R);
  d.frame_label = dalloc<int>(c, (size_t)R * kp.fcap);
  if (kp.hi) {
    d.hi_m = dalloc<int4>(c, kp.hi_nm);
    d.hi_w = dalloc<float>(c, kp.hi_nm);
    d.hi_excl = dalloc<uint32_t>(c, nlam);
    d.hi_M = dalloc<double>(c, (size_t)R * G * 10);
    d.hi_F = dalloc<float>(c, (size_t)R * nlam * 3);
    d.hi_dvdl = dalloc<double>(c, (size_t)R * C);
    if (!d.hi_dvdl) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
  }
  if (kp.P) {
    const int P = kp.P, L = kp.remd_total / P;
    d.lvl_d1 = dalloc<double>(c, (size_t)P * C);
    d.lvl_dG = dalloc<double>(c, (size_t)P * G * 3);
    d.remd_label = dalloc<int>(c, R);
    d.remd_rows = dalloc<double>(c, (size_t)R * (P + 1));
    d.remd_holder = dalloc<int>(c, kp.remd_total);
    d.remd_newlab = dalloc<int>(c, kp.remd_total);
    d.remd_att = dalloc<long long>(c, (size_t)L * (P - 1));
    d.remd_acc = dalloc<long long>(c, (size_t)L * (P - 1));
    if (!d.remd_acc) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
  }
  for (void *p : {(void *)d.xyzq, kp.pair_mode ? (void *)d.cl_j : (void *)d.nbl, (void *)d.grid, (void *)d.cgrid, (void *)d.flags, (void *)d.seed})
    if (!p) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
  if (c.allocations.size() < 40) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }

  // ---- uploads -----------------------------------------------------------------------
  std::vector<float4> hx(RN), hv(RN);
  std::vector<int2> hm(RN);
  std::vector<int> hperm((size_t)R * N);
  for (int r = 0; r < R; ++r) {
    const float *P = prm->pos_replicas ? prm->pos_replicas + (size_t)r * N * 3 : sys->pos;
    const float *Vv = prm->vel_replicas ? prm->vel_replicas + (size_t)r * N * 3 : sys->vel;
    if (prm->pos_replicas && !finite_arr(P, 3 * (size_t)N)) return bad("non-finite pos_replicas");
    if (prm->vel_replicas && !finite_arr(Vv, 3 * (size_t)N)) return bad("non-finite vel_replicas");
    for (int i = 0; i < N; ++i) {
      const size_t idx = (size_t)r * kp.Nst + i;
      const float q = lslot[i] >= 0 ? 0.0f : sys->charge[i];
      hx[idx] = make_float4(P[3 * i], P[3 * i + 1], P[3 * i + 2], q);
      const float m = sys->mass[i];
      const float invm = m > 0.0f ? 1.0f / m : 0.0f;
      if (Vv && m > 0.0f) hv[idx] = make_float4(Vv[3 * i], Vv[3 * i + 1], Vv[3 * i + 2], invm);
      else hv[idx] = make_float4(0.f, 0.f, 0.f, invm);
      hm[idx] = make_int2(i, sys->type[i] | ((lslot[i] + 1) << 8));
      hperm[(size_t)r * N + i] = i;
    }
  }
  std::vector<float2> lj((size_t)T * T);
  for (int t = 0; t < T * T; ++t) lj[t] = make_float2((float)(6.0 * sys->c6[t]), (float)(12.0 * sys->c12[t]));
  std::vector<float> bsp;
  for (int dd = 0; dd < 3; ++dd) bsp_moduli(kp.K[dd], bsp);
  std::vector<double> lam0((size_t)R * C, 0.0);
  if (prm->lambda0) std::copy(prm->lambda0, prm->lambda0 + (size_t)R * C, lam0.begin());
  c.h_seed.assign(prm->replica_seed, prm->replica_seed + R);
  c.h_pH.assign(prm->pH, prm->pH + R);
  c.h_d1.assign((size_t)R * C, 0.0);
  c.h_dG.assign((size_t)R * G * 3, 0.0);
  c.h_dw.resize((size_t)R * C * 4);
  for (size_t k = 0; k < (size_t)R * C; ++k) {
    c.h_dw[4 * k] = 0.0; c.h_dw[4 * k + 1] = 1.0;
    c.h_dw[4 * k + 2] = c.h_dw[4 * k + 3] = prm->barrier;
  }
  c.h_c_group.assign(C, 0);
  c.h_c_lp.assign(C, -1);
  for (int g = 0; g < G; ++g) {
    for (int k = c.h_cptr[g]; k < c.h_cptr[g + 1]; ++k) c.h_c_group[k] = g;
    if (c.h_group_kind[g] == 3) c.h_c_lp[c.h_cptr[g] + 1] = c.h_cptr[g];
  }
  c.h_cens.assign((size_t)R * G * 2, 0);

#define UP(dst, src, n) CK(cudaMemcpy(dst, src, sizeof(*(src)) * (n), cudaMemcpyHostToDevice))
  {
    auto up = [&]() -> cph_status {
      UP(d.xyzq, hx.data(), RN); UP(d.vel, hv.data(), RN); UP(d.meta, hm.data(), RN);
      UP(d.iperm, hperm.data(), (size_t)R * N);
      UP(d.excl_ptr, c.h_excl_ptr.data(), N + 1);
      if (!c.h_excl_idx.empty()) UP(d.excl_idx, c.h_excl_idx.data(), c.h_excl_idx.size());
      UP(d.ljtab, lj.data(), lj.size());
      UP(d.bsp, bsp.data(), bsp.size());
      if (G) {
        UP(d.g_kind, c.h_group_kind.data(), G); UP(d.g_ptr, c.h_group_ptr.data(), G + 1);
        UP(d.g_atoms, c.h_group_atoms.data(), nlam); UP(d.g_cptr, c.h_cptr.data(), G + 1);
        UP(d.g_q, c.h_state_q.data(), 4 * (size_t)nlam); UP(d.vmm, sys->vmm, 36 * (size_t)G);
        std::vector<int> kg(nlam);
        for (int g = 0; g < G; ++g)
          for (int k = c.h_group_ptr[g]; k < c.h_group_ptr[g + 1]; ++k) kg[k] = g;
        UP(d.k_group, kg.data(), nlam);
      }
      if (kp.hi) {
        UP(d.hi_m, hi_m.data(), hi_m.size());
        UP(d.hi_w, hi_w.data(), hi_w.size());
        std::vector<uint32_t> mask(nlam, 0u);
        for (int g = 0; g < G; ++g)
          for (int i = c.h_group_ptr[g]; i < c.h_group_ptr[g + 1]; ++i) {
            const int a = c.h_group_atoms[i];
            for (int j = c.h_group_ptr[g]; j < c.h_group_ptr[g + 1]; ++j) {
              const int b = c.h_group_atoms[j];
              for (int e = c.h_excl_ptr[a]; e < c.h_excl_ptr[a + 1]; ++e)
                if (c.h_excl_idx[e] == b) mask[i] |= 1u << (j - c.h_group_ptr[g]);
            }
          }
        UP(d.hi_excl, mask.data(), nlam);
      }
      if (C) {
        UP(d.lam, lam0.data(), (size_t)R * C);
        UP(d.dw, c.h_dw.data(), c.h_dw.size());
        UP(d.c_group, c.h_c_group.data(), C);
        UP(d.c_lp, c.h_c_lp.data(), C);
      }
      UP(d.seed, c.h_seed.data(), R);
      return CPH_OK;
    };
    cph_status st = up();
    if (st != CPH_OK) return fail_create(ctx, st);
  }
#undef UP
  {
    std::vector<int> all(R);
    for (int r = 0; r < R; ++r) all[r] = r;
    cph_status st = kp.P ? run_pfc_levels(c, labels0) : run_pfc_many(c, all);
    if (st != CPH_OK) return fail_create(ctx, st);
  }
  // cuFFT plans (batched over replicas)
  {
    int n3[3] = {kp.K[0], kp.K[1], kp.K[2]};
    if (cufftPlanMany(&c.plan_r2c, 3, n3, nullptr, 1, kp.K3, nullptr, 1, kp.Kc, kp.fft64 ? CUFFT_D2Z : CUFFT_R2C, R) !=
            CUFFT_SUCCESS ||
        cufftPlanMany(&c.plan_c2r, 3, n3, nullptr, 1, kp.Kc, nullptr, 1, kp.K3, kp.fft64 ? CUFFT_Z2D : CUFFT_C2R, R) !=
            CUFFT_SUCCESS) {
      c.err = "cufftPlanMany failed";
      return fail_create(ctx, CPH_E_CUDA);
    }
  }
  c.host_step = 0;
  c.launches += launch_influence(c, c.stream);
  cph_status st = evaluate_here(c, true);
  if (st == CPH_OK) st = check_flags(c);
  // a denser-than-average region overflowed the list capacity: grow it once (with margin)
  // and rebuild; an overflow during stepping is reported by the next call instead
  if (st == CPH_E_STATE && (c.cap_grow > (size_t)kp.cap || c.clcap_grow > (size_t)kp.clcap)) {
    auto release = [&](void *old) {
      c.allocations.erase(std::remove(c.allocations.begin(), c.allocations.end(), old), c.allocations.end());
      if (c.dev_free) c.dev_free(old, c.alloc_ctx); else cudaFree(old);
    };
    if (c.cap_grow > (size_t)kp.cap) {
      kp.cap = (int)((c.cap_grow * 5 / 4 + 64 + 7) / 8 * 8);
      if (kp.pair_mode == 0) {
        release(d.nbl);
        d.nbl = dalloc<uint32_t>(c, RN * kp.cap);
        if (!d.nbl) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
      } else {
        release(d.lam_nbl);
        d.lam_nbl = dalloc<uint32_t>(c, std::max<size_t>(1, (size_t)R * nlam * kp.cap));
        if (!d.lam_nbl) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
      }
    }
    if (c.clcap_grow > (size_t)kp.clcap) {
      kp.clcap = (int)(c.clcap_grow * 5 / 4 + 64);
      release(d.cl_j);
      release(d.cl_m);
      d.cl_j = dalloc<uint32_t>(c, (size_t)R * kp.nsc * kp.clcap);
      d.cl_m = dalloc<uint4>(c, (size_t)R * kp.nsc * kp.clcap);
      if (!d.cl_j || !d.cl_m) { c.err = "device allocation failed"; return fail_create(ctx, CPH_E_OOM); }
    }
    const int zero[FLAG_COUNT] = {0};
    if (cudaMemcpy(d.flags, zero, sizeof(zero), cudaMemcpyHostToDevice) != cudaSuccess) {
      c.err = "flag reset failed";
      return fail_create(ctx, CPH_E_CUDA);
    }
    c.err.clear();
    st = evaluate_here(c, true);
    if (st == CPH_OK) st = check_flags(c);
  }
  // the nstlist-block graph is captured now (capture records, runs nothing), so the first
  // full block of a cph_step call replays it instead of paying capture + instantiation
  if (st == CPH_OK) st = capture_block(c);
  if (st != CPH_OK) {
    cph_status s2 = st;
    if (c.plan_r2c) cufftDestroy(c.plan_r2c);
    if (c.plan_c2r) cufftDestroy(c.plan_c2r);
    return fail_create(ctx, s2);
  }
  *out = ctx;
  return CPH_OK;
}

static void sub_destroy(SubCtx *ctx) {
  if (!ctx) return;
  Ctx &c = ctx->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  if (c.tl) { tl_print(c); cudaFree(c.tl->stamps); delete c.tl; c.tl = nullptr; }
  if (c.graph_block) cudaGraphExecDestroy(c.graph_block);
  if (c.plan_r2c) cufftDestroy(c.plan_r2c);
  if (c.plan_c2r) cufftDestroy(c.plan_c2r);
  free_all(c);
  if (c.h_bad) cudaFreeHost(c.h_bad);
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  if (c.ev_join) cudaEventDestroy(c.ev_join);
  if (c.ev_gather) cudaEventDestroy(c.ev_gather);
  if (c.stream_pme) cudaStreamDestroy(c.stream_pme);
  if (c.stream_nb) cudaStreamDestroy(c.stream_nb);
  if (c.ev_fork2) cudaEventDestroy(c.ev_fork2);
  if (c.ev_join2) cudaEventDestroy(c.ev_join2);
  if (c.own_stream) cudaStreamDestroy(c.stream);
  delete ctx;
}

static int32_t sub_n_coords(const SubCtx *ctx) { return ctx ? ctx->c.kp.C : -1; }
static int32_t sub_n_atoms(const SubCtx *ctx) { return ctx ? ctx->c.kp.N : -1; }
static int64_t sub_current_step(const SubCtx *ctx) { return ctx ? ctx->c.host_step : -1; }
static int64_t sub_launch_count(const SubCtx *ctx) { return ctx ? ctx->c.launches : -1; }

static cph_status sub_set_pH(SubCtx *ctx, int32_t replica, double pH) {
  CPH_NVTX("cph_set_pH");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, replica);
  if (st) return st;
  if (!std::isfinite(pH)) { c.err = "non-finite pH"; return CPH_E_INVALID; }
  if (c.kp.P) { c.err = "pH is set through the replica-exchange labels (cph_set_labels)"; return CPH_E_STATE; }
  cudaSetDevice(c.device);
  CK(cudaStreamSynchronize(c.stream));
  const double old = c.h_pH[replica];
  c.h_pH[replica] = pH;
  st = run_pfc(c, replica);
  if (st != CPH_OK) {
    c.h_pH[replica] = old;
    return st;
  }
  // dV_bias/dlambda and E_bias at the unchanged lambda under the new pH tables, so the next
  // half kick and the getters see the new Hamiltonian (the Coulomb part is unchanged)
  c.launches += launch_bias_refresh(c, c.stream);
  CK(cudaGetLastError());
  return check_flags(c);
}

// steps host_step -> end as one asynchronous segment (graphs of nstlist steps where aligned)
static cph_status run_segment(Ctx &c, long long end) {
  k_set_end<<<1, 1, 0, c.stream>>>(c.d.end_step, end);
  int k = 1;
  k += launch_lambda_open(c, c.stream);
  const int nl = c.kp.nstlist;
  while (c.host_step < end) {
    const long long remaining = end - c.host_step;
    if (c.host_step % nl == 0 && remaining >= nl) {
      cph_status st = capture_block(c);
      if (st) return st;
      CK(cudaGraphLaunch(c.graph_block, c.stream));
      if (c.tl) tl_collect(c);
      k += c.graph_block_kernels;
      c.host_step += nl;
    } else {
      k += enqueue_step(c, (c.host_step + 1) % nl == 0, getenv("CPH_ONE_STREAM") == nullptr);
      c.host_step += 1;
    }
  }
  k += launch_close(c, c.stream, 1);
  c.launches += k;
  CK(cudaGetLastError());
  return CPH_OK;
}

// ---- DBO controllers (R23-R26) -----------------------------
static double well_decide(const DboConfig &b, double shift, double n, double n_near, double sum_near, double ideal) {
  if (n <= 0.0 || n_near <= 0.0 || !(n_near / n > b.residency)) return shift;
  const double diff = ideal - sum_near / n_near;
  if (!(std::fabs(diff) > b.tol)) return shift;
  return std::min(b.cap, std::max(-b.cap, shift + b.gain * diff));
}

static double barrier_decide(const DboConfig &b, double h, double n, double n_trans) {
  if (n <= 0.0) return h;
  const double frac = n_trans / n;
  if (frac < b.target - b.target_tol) return std::max(b.bmin, h - b.bstep);
  if (frac > b.target + b.target_tol) return std::min(b.bmax, h + b.bstep);
  return h;
}

// End of step S = host_step: run the due block rules for every replica, log and censor the
// adjusted sites, refresh their PFC and re-evaluate the forces at the unchanged state so
// step S+1 starts on the new bias.
static cph_status dbo_block_end(Ctx &c) {
  CPH_NVTX("dbo_block_end");
  const KParams &kp = c.kp;
  const DboConfig &b = c.dbo;
  const long long S = c.host_step;
  const bool do_well = b.well && S % b.well_steps == 0;
  const bool do_bar = b.barrier && S % b.barrier_steps == 0;
  if (!do_well && !do_bar) return CPH_OK;
  const int R = kp.R, C = kp.C, G = kp.G;
  std::vector<double> wst((size_t)R * C * 5), bst((size_t)R * C * 4);
  CK(cudaStreamSynchronize(c.stream));
  if (do_well) {
    CK(cudaMemcpy(wst.data(), c.d.dbo_well, sizeof(double) * wst.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemset(c.d.dbo_well, 0, sizeof(double) * wst.size()));
  }
  if (do_bar) {
    CK(cudaMemcpy(bst.data(), c.d.dbo_bar, sizeof(double) * bst.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemset(c.d.dbo_bar, 0, sizeof(double) * bst.size()));
  }
  std::vector<std::vector<char>> changed_all(R, std::vector<char>(G, 0));
  std::vector<int> reps;
  for (int r = 0; r < R; ++r) {
    std::vector<char> &changed = changed_all[r];
    auto log = [&](int k, int kind, double o, double n) {
      c.events.push_back(cph_dbo_event{S, r, k, kind, 0, o, n});
      changed[c.h_c_group[k]] = 1;
    };
    double *dw = c.h_dw.data() + (size_t)r * C * 4;
    if (do_well)
      for (int k = 0; k < C; ++k) {
        const double *a = wst.data() + ((size_t)r * C + k) * 5;
        double *w = dw + 4 * k;
        const double a0 = well_decide(b, w[0], a[0], a[1], a[2], 0.0);
        const double a1 = 1.0 + well_decide(b, w[1] - 1.0, a[0], a[3], a[4], 1.0);
        if (a0 != w[0]) { log(k, CPH_DBO_WELL0, w[0], a0); w[0] = a0; }
        if (a1 != w[1]) { log(k, CPH_DBO_WELL1, w[1], a1); w[1] = a1; }
      }
    if (do_bar)
      for (int k = 0; k < C; ++k) {
        const double *a = bst.data() + ((size_t)r * C + k) * 4;
        double *w = dw + 4 * k;
        if (c.h_c_lp[k] < 0) {
          const double h = barrier_decide(b, w[2], a[0], a[1]);
          if (h != w[2]) { log(k, CPH_DBO_BARRIER, w[2], h); w[2] = w[3] = h; }
        } else {
          const double hp = barrier_decide(b, w[2], a[0], a[1]);
          const double hd = barrier_decide(b, w[3], a[2], a[3]);
          if (hp != w[2]) { log(k, CPH_DBO_BARRIER_T_PROT, w[2], hp); w[2] = hp; }
          if (hd != w[3]) { log(k, CPH_DBO_BARRIER_T_DEPROT, w[3], hd); w[3] = hd; }
        }
      }
    bool rc = false;
    for (int g = 0; g < G; ++g)
      if (changed[g]) {
        rc = true;
        long long *w = c.h_cens.data() + ((size_t)r * G + g) * 2;   // (from, until]
        if (!(S < w[1])) w[0] = S;
        w[1] = S + b.censor_steps;
      }
    if (rc) reps.push_back(r);
  }
  if (reps.empty()) return CPH_OK;
  if (cph_status st = run_pfc_many(c, reps, &changed_all)) return st;
  CK(cudaMemcpy(c.d.dw, c.h_dw.data(), sizeof(double) * c.h_dw.size(), cudaMemcpyHostToDevice));
  if (G) CK(cudaMemcpy(c.d.cens, c.h_cens.data(), sizeof(long long) * c.h_cens.size(), cudaMemcpyHostToDevice));
  return evaluate_here(c, false);          // block ends are multiples of nstlist: the list is fresh
}

static long long next_dbo_boundary(const Ctx &c) {
  long long nb = LLONG_MAX;
  const long long s = c.host_step;
  if (c.dbo.well) nb = std::min(nb, (s / c.dbo.well_steps + 1) * c.dbo.well_steps);
  if (c.dbo.barrier) nb = std::min(nb, (s / c.dbo.barrier_steps + 1) * c.dbo.barrier_steps);
  return nb;
}

static cph_status sub_step(SubCtx *ctx, int64_t n_steps) {
  CPH_NVTX("cph_step");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  if (n_steps < 0) { c.err = "n_steps < 0"; return CPH_E_INVALID; }
  if (n_steps == 0) return CPH_OK;
  cudaSetDevice(c.device);
  const long long end = c.host_step + n_steps;
  while (c.host_step < end) {
    const long long seg = c.kp.dbo_on ? std::min(end, next_dbo_boundary(c)) : end;
    cph_status st = run_segment(c, seg);
    if (st) return st;
    if (c.kp.dbo_on && (st = dbo_block_end(c))) return st;
  }
  return CPH_OK;
}

static cph_status sub_sync(SubCtx *ctx) {
  CPH_NVTX("cph_sync");
  if (!ctx) return CPH_E_INVALID;
  cudaSetDevice(ctx->c.device);
  return check_flags(ctx->c);
}

static cph_status sub_get_lambdas(SubCtx *ctx, int32_t r, double *lam, double *vel) {
  CPH_NVTX("cph_get_lambdas");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t C = c.kp.C;
  if (lam && C) CK(cudaMemcpy(lam, c.d.lam + r * C, sizeof(double) * C, cudaMemcpyDeviceToHost));
  if (vel && C) CK(cudaMemcpy(vel, c.d.lamv + r * C, sizeof(double) * C, cudaMemcpyDeviceToHost));
  return CPH_OK;
}

static cph_status sub_get_dvdl(SubCtx *ctx, int32_t r, double *coul, double *bias) {
  CPH_NVTX("cph_get_dvdl");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t C = c.kp.C;
  if (coul && C) CK(cudaMemcpy(coul, c.d.dvdl_coul + r * C, sizeof(double) * C, cudaMemcpyDeviceToHost));
  if (bias && C) CK(cudaMemcpy(bias, c.d.dvdl_bias + r * C, sizeof(double) * C, cudaMemcpyDeviceToHost));
  return CPH_OK;
}

static cph_status sub_get_bias_params(SubCtx *ctx, int32_t r, double *d1) {
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st) return st;
  if (d1 && c.kp.P) {          // labels may have moved on the device
    if ((st = sub_sync(ctx))) return st;
    if (c.kp.C) CK(cudaMemcpy(d1, c.d.d1 + (size_t)r * c.kp.C, sizeof(double) * c.kp.C, cudaMemcpyDeviceToHost));
    return CPH_OK;
  }
  if (d1) std::copy(c.h_d1.begin() + (size_t)r * c.kp.C, c.h_d1.begin() + (size_t)(r + 1) * c.kp.C, d1);
  return CPH_OK;
}

static cph_status sub_get_energies(SubCtx *ctx, int32_t r, double *e) {
  CPH_NVTX("cph_get_energies");
  if (!ctx || !e) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t off = ((size_t)(c.host_step & 1) * c.kp.R + r) * kNE;
  CK(cudaMemcpy(e, c.d.erec + off, sizeof(double) * kNE, cudaMemcpyDeviceToHost));
  double tot = 0.0;
  for (int k = 0; k < CPH_E_TOTAL; ++k) tot += e[k];
  e[CPH_E_TOTAL] = tot;
  return CPH_OK;
}

static cph_status sub_get_frames_ex(SubCtx *ctx, int32_t r, float *buf, uint8_t *censored, int64_t *steps, int32_t *labels,
                             int64_t cap, int64_t *n_frames, int64_t *n_dropped) {
  CPH_NVTX("cph_get_frames_ex");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  if (cap < 0) { c.err = "cap < 0"; return CPH_E_INVALID; }
  const KParams &kp = c.kp;
  long long total = 0;
  CK(cudaMemcpy(&total, c.d.frame_total + r, sizeof(long long), cudaMemcpyDeviceToHost));
  const long long avail = std::min<long long>(total, kp.fcap);
  const long long take = std::min<long long>(avail, cap);
  std::vector<float> all((size_t)kp.fcap * kp.C);
  std::vector<unsigned char> cens((size_t)kp.fcap * kp.C);
  std::vector<long long> fst(kp.fcap);
  std::vector<int> flab(kp.fcap);
  CK(cudaMemcpy(flab.data(), c.d.frame_label + (size_t)r * kp.fcap, sizeof(int) * kp.fcap, cudaMemcpyDeviceToHost));
  if (kp.C) {
    CK(cudaMemcpy(all.data(), c.d.frames + (size_t)r * kp.fcap * kp.C, sizeof(float) * all.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cens.data(), c.d.frame_cens + (size_t)r * kp.fcap * kp.C, cens.size(), cudaMemcpyDeviceToHost));
  }
  CK(cudaMemcpy(fst.data(), c.d.frame_step + (size_t)r * kp.fcap, sizeof(long long) * kp.fcap, cudaMemcpyDeviceToHost));
  // oldest retained frame index = total - avail; we return the newest `take` frames in order
  const long long first = total - take;
  for (long long f = 0; f < take; ++f) {
    const long long slot = (first + f) % kp.fcap;
    for (int k = 0; k < kp.C; ++k) {
      if (buf) buf[f * kp.C + k] = all[(size_t)slot * kp.C + k];
      if (censored) censored[f * kp.C + k] = cens[(size_t)slot * kp.C + k];
    }
    if (steps) steps[f] = fst[slot];
    if (labels) labels[f] = flab[slot];
  }
  if (n_frames) *n_frames = take;
  if (n_dropped) *n_dropped = total - take;
  const long long zero = 0;
  CK(cudaMemcpy(c.d.frame_total + r, &zero, sizeof(long long), cudaMemcpyHostToDevice));
  return CPH_OK;
}

static cph_status sub_get_frames(SubCtx *ctx, int32_t r, float *buf, int64_t cap, int64_t *n_frames, int64_t *n_dropped) {
  return sub_get_frames_ex(ctx, r, buf, nullptr, nullptr, nullptr, cap, n_frames, n_dropped);
}

static cph_status need_remd(Ctx &c) {
  if (!c.kp.P) { c.err = "replica exchange is off (n_ph_levels = 0)"; return CPH_E_STATE; }
  return CPH_OK;
}

static cph_status sub_exchange_energies(SubCtx *ctx, double *rows) {
  CPH_NVTX("cph_exchange_energies");
  if (!ctx || !rows) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  if (cph_status st = need_remd(c)) return st;
  cudaSetDevice(c.device);
  c.launches += launch_remd_energy(c, c.stream, rows);
  CK(cudaGetLastError());
  return CPH_OK;
}

static cph_status sub_exchange_apply(SubCtx *ctx, const double *rows_all, uint64_t seed, int64_t attempt) {
  CPH_NVTX("cph_exchange_apply");
  if (!ctx || !rows_all || attempt < 0) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  if (cph_status st = need_remd(c)) return st;
  cudaSetDevice(c.device);
  c.launches += launch_remd_apply(c, c.stream, rows_all, seed, attempt);
  c.launches += launch_bias_refresh(c, c.stream);
  CK(cudaGetLastError());
  return CPH_OK;
}

static cph_status sub_exchange(SubCtx *ctx, uint64_t seed, int64_t attempt) {
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  if (cph_status st = need_remd(c)) return st;
  if (c.kp.remd_total != c.kp.R) { c.err = "cph_exchange needs every replica in this context"; return CPH_E_STATE; }
  cph_status st = sub_exchange_energies(ctx, c.d.remd_rows);
  return st ? st : sub_exchange_apply(ctx, c.d.remd_rows, seed, attempt);
}

static cph_status sub_get_labels(SubCtx *ctx, int32_t *labels) {
  if (!ctx || !labels) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = need_remd(c);
  if (st || (st = sub_sync(ctx))) return st;
  CK(cudaMemcpy(labels, c.d.remd_label, sizeof(int) * c.kp.R, cudaMemcpyDeviceToHost));
  return CPH_OK;
}

static cph_status sub_set_labels(SubCtx *ctx, const int32_t *labels) {
  CPH_NVTX("cph_set_labels");
  if (!ctx || !labels) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = need_remd(c);
  if (st) return st;
  for (int r = 0; r < c.kp.R; ++r)
    if (labels[r] < 0 || labels[r] >= c.kp.P) { c.err = "label out of range"; return CPH_E_INVALID; }
  if (!labels_form_ladders(labels, c.kp.R, c.kp.remd_first, c.kp.P)) {
    c.err = "each pH ladder held by this context must carry every level exactly once";
    return CPH_E_INVALID;
  }
  cudaSetDevice(c.device);
  CK(cudaStreamSynchronize(c.stream));
  std::vector<int> lab(labels, labels + c.kp.R);
  if ((st = run_pfc_levels(c, lab))) return st;
  c.launches += launch_bias_refresh(c, c.stream);
  return check_flags(c);
}

static cph_status sub_get_exchange_stats(SubCtx *ctx, int64_t *attempts, int64_t *accepts) {
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = need_remd(c);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t n = (size_t)(c.kp.remd_total / c.kp.P) * (c.kp.P - 1);
  if (attempts) CK(cudaMemcpy(attempts, c.d.remd_att, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  if (accepts) CK(cudaMemcpy(accepts, c.d.remd_acc, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  return CPH_OK;
}

static cph_status sub_get_dbo_params(SubCtx *ctx, int32_t r, double *p) {
  if (!ctx || !p) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st) return st;
  std::copy(c.h_dw.begin() + (size_t)r * c.kp.C * 4, c.h_dw.begin() + (size_t)(r + 1) * c.kp.C * 4, p);
  return CPH_OK;
}

static cph_status sub_set_dbo_params(SubCtx *ctx, int32_t r, const double *p) {
  CPH_NVTX("cph_set_dbo_params");
  if (!ctx || !p) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st) return st;
  const int C = c.kp.C;
  if (!finite_arr(p, (size_t)C * 4)) { c.err = "non-finite DBO parameter"; return CPH_E_INVALID; }
  for (int k = 0; k < C; ++k) {
    const double *w = p + 4 * k;
    if (std::fabs(w[0]) > 0.2 || std::fabs(w[1] - 1.0) > 0.2 || !(w[2] > 0.0 && w[2] <= 100.0) ||
        !(w[3] > 0.0 && w[3] <= 100.0) || (c.h_c_lp[k] < 0 && w[2] != w[3])) {
      c.err = "DBO parameters out of range (|a0| <= 0.2, |a1-1| <= 0.2, 0 < h <= 100, lambda_p: h_prot == h_deprot)";
      return CPH_E_INVALID;
    }
  }
  cudaSetDevice(c.device);
  CK(cudaStreamSynchronize(c.stream));
  std::copy(p, p + (size_t)C * 4, c.h_dw.begin() + (size_t)r * C * 4);
  if (C) CK(cudaMemcpy(c.d.dw + (size_t)r * C * 4, p, sizeof(double) * C * 4, cudaMemcpyHostToDevice));
  if ((st = run_pfc(c, r))) return st;
  if ((st = evaluate_here(c, false))) return st;     // positions unchanged: the list stands
  return check_flags(c);
}

static cph_status sub_get_dbo_stats(SubCtx *ctx, int32_t r, double *well, double *barrier) {
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t C = c.kp.C;
  if (well && C) CK(cudaMemcpy(well, c.d.dbo_well + r * C * 5, sizeof(double) * C * 5, cudaMemcpyDeviceToHost));
  if (barrier && C) CK(cudaMemcpy(barrier, c.d.dbo_bar + r * C * 4, sizeof(double) * C * 4, cudaMemcpyDeviceToHost));
  return CPH_OK;
}

static cph_status sub_get_forces(SubCtx *ctx, int32_t r, float *f, float *phi) {
  CPH_NVTX("cph_get_forces");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const KParams &kp = c.kp;
  const size_t N = kp.N, base = (size_t)r * kp.Nst;
  std::vector<float4> nb(N), rec(N), xq(N);
  std::vector<int2> meta(N);
  std::vector<double> plam(kp.nlam), qlam(kp.nlam);
  CK(cudaMemcpy(nb.data(), c.d.f_nb + base, sizeof(float4) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rec.data(), c.d.f_rec + base, sizeof(float4) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(xq.data(), c.d.xyzq + base, sizeof(float4) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(meta.data(), c.d.meta + base, sizeof(int2) * N, cudaMemcpyDeviceToHost));
  if (kp.nlam) {
    CK(cudaMemcpy(plam.data(), c.d.phi_lam + (size_t)r * kp.nlam, sizeof(double) * kp.nlam, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(qlam.data(), c.d.qlam + (size_t)r * kp.nlam, sizeof(double) * kp.nlam, cudaMemcpyDeviceToHost));
  }
  double Q = kp.Q_fixed;
  for (double q : qlam) Q += q;
  const double V = kp.Ld[0] * kp.Ld[1] * kp.Ld[2];
  const double phinet = -kPi * Q / (V * kp.beta_d * kp.beta_d);
  const double selfc = -2.0 * kp.beta_d / std::sqrt(kPi);
  for (size_t s = 0; s < N; ++s) {
    const int o = meta[s].x;
    const int ls = (meta[s].y >> 8) - 1;
    if (f) {
      f[3 * o] = nb[s].x + rec[s].x;
      f[3 * o + 1] = nb[s].y + rec[s].y;
      f[3 * o + 2] = nb[s].z + rec[s].z;
    }
    if (phi) {
      if (ls >= 0) phi[o] = (float)(plam[ls] + phinet);   // kernel phi excludes the net-charge term
      else phi[o] = (float)((double)nb[s].w + (double)rec[s].w + selfc * xq[s].w + phinet);
    }
  }
  return CPH_OK;
}

static cph_status sub_get_positions(SubCtx *ctx, int32_t r, float *pos, float *vel) {
  CPH_NVTX("cph_get_positions");
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const size_t N = c.kp.N, base = (size_t)r * c.kp.Nst;
  std::vector<float4> xq(N), v(N);
  std::vector<int2> meta(N);
  CK(cudaMemcpy(xq.data(), c.d.xyzq + base, sizeof(float4) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(v.data(), c.d.vel + base, sizeof(float4) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(meta.data(), c.d.meta + base, sizeof(int2) * N, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < N; ++s) {
    const int o = meta[s].x;
    if (pos) { pos[3 * o] = xq[s].x; pos[3 * o + 1] = xq[s].y; pos[3 * o + 2] = xq[s].z; }
    if (vel) { vel[3 * o] = v[s].x; vel[3 * o + 1] = v[s].y; vel[3 * o + 2] = v[s].z; }
  }
  return CPH_OK;
}


// Pair-list decoding for the getters (host side).  The device list of replica r is copied
// once; row(slot) gives the original indices of every entry the pair kernel evaluates for
// that sorted slot (padding entries, which point at the atom itself, are skipped).
struct ListHost {
  std::vector<int> nnb;
  std::vector<int2> meta;
  std::vector<int> iperm;
  std::vector<uint32_t> nbl;
  std::vector<int64_t> rp;       // cluster mode: directed partner slots of every slot (CSR)
  std::vector<int> cols;
};

static cph_status fetch_list(Ctx &c, int r, ListHost &h) {
  const KParams &kp = c.kp;
  const size_t N = kp.N, base = (size_t)r * kp.Nst;
  h.meta.resize(N);
  h.iperm.resize(N);
  CK(cudaMemcpy(h.meta.data(), c.d.meta + base, sizeof(int2) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h.iperm.data(), c.d.iperm + (size_t)r * N, sizeof(int) * N, cudaMemcpyDeviceToHost));
  if (kp.pair_mode == 1) {
    // every set mask bit of every entry is one pair the kernel evaluates, acting on both atoms
    const size_t ns = kp.nsc, sb = (size_t)r * ns;
    std::vector<int> n(ns), first(ns), ni(ns);
    std::vector<uint32_t> cj(ns * kp.clcap);
    std::vector<uint4> cm(ns * kp.clcap);
    CK(cudaMemcpy(n.data(), c.d.cl_n + sb, sizeof(int) * ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(first.data(), c.d.sc_first + sb, sizeof(int) * ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ni.data(), c.d.sc_ni + sb, sizeof(int) * ns, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cj.data(), c.d.cl_j + sb * kp.clcap, sizeof(uint32_t) * cj.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cm.data(), c.d.cl_m + sb * kp.clcap, sizeof(uint4) * cm.size(), cudaMemcpyDeviceToHost));
    std::vector<int> pi, pj;
    for (size_t id = 0; id < ns; ++id) {
      if (!ni[id]) continue;
      for (int e = 0; e < std::min(n[id], kp.clcap); ++e) {
        const size_t k = id * kp.clcap + e;
        const uint32_t w[4] = {cm[k].x, cm[k].y, cm[k].z, cm[k].w};
        const int J = (int)(cj[k] & kClJMask);
        for (int s = 0; s < 4; ++s)
          for (int bit = 0; bit < 32; ++bit)
            if ((w[s] >> bit) & 1u) {
              pi.push_back(first[id] + 8 * s + (bit & 7));
              pj.push_back(4 * J + (bit >> 3));
            }
      }
    }
    h.rp.assign(N + 1, 0);
    for (size_t k = 0; k < pi.size(); ++k) { ++h.rp[pi[k] + 1]; ++h.rp[pj[k] + 1]; }
    for (size_t k = 0; k < N; ++k) h.rp[k + 1] += h.rp[k];
    h.cols.resize(h.rp[N]);
    std::vector<int64_t> fill(h.rp.begin(), h.rp.end() - 1);
    for (size_t k = 0; k < pi.size(); ++k) { h.cols[fill[pi[k]]++] = pj[k]; h.cols[fill[pj[k]]++] = pi[k]; }
    return CPH_OK;
  }
  h.nnb.resize(N);
  h.nbl.resize((size_t)kp.cap * kp.Nst);
  CK(cudaMemcpy(h.nnb.data(), c.d.nnb + base, sizeof(int) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h.nbl.data(), c.d.nbl + (size_t)r * kp.cap * kp.Nst, sizeof(uint32_t) * h.nbl.size(),
                cudaMemcpyDeviceToHost));
  return CPH_OK;
}

template <class F>
static void list_row(const Ctx &c, const ListHost &h, int slot, F emit) {
  const KParams &kp = c.kp;
  if (kp.pair_mode == 1) {
    for (int64_t k = h.rp[slot]; k < h.rp[slot + 1]; ++k) emit(h.meta[h.cols[k]].x);
    return;
  }
  for (int k = 0; k < std::min(h.nnb[slot], kp.cap); ++k) {
    const int j = (int)(h.nbl[((size_t)(k / 8) * kp.Nst + slot) * 8 + (k % 8)] & kEntryJMask);
    if (j != slot) emit(h.meta[j].x);
  }
}

static cph_status decode_directed(Ctx &c, int r, std::vector<std::pair<int, int>> &out) {
  ListHost h;
  if (cph_status st = fetch_list(c, r, h)) return st;
  out.clear();
  for (int i = 0; i < c.kp.N; ++i) {
    const int oi = h.meta[i].x;
    list_row(c, h, i, [&](int oj) { out.emplace_back(oi, oj); });
  }
  return CPH_OK;
}


static cph_status sub_get_pairlist_rows(SubCtx *ctx, int32_t r, const int32_t *atoms, int32_t n_atoms, int32_t *row_ptr,
                                 int32_t *cols, int64_t cap) {
  CPH_NVTX("cph_get_pairlist_rows");
  if (!ctx || !atoms || !row_ptr || n_atoms < 0 || cap < 0) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  for (int k = 0; k < n_atoms; ++k)
    if (atoms[k] < 0 || atoms[k] >= c.kp.N) { c.err = "atom index out of range"; return CPH_E_INVALID; }
  ListHost h;
  if ((st = fetch_list(c, r, h))) return st;
  int64_t n = 0;
  row_ptr[0] = 0;
  std::vector<int> row;
  for (int k = 0; k < n_atoms; ++k) {
    row.clear();
    list_row(c, h, h.iperm[atoms[k]], [&](int oj) { row.push_back(oj); });
    std::sort(row.begin(), row.end());
    for (int oj : row) {
      if (cols && n < cap) cols[n] = oj;
      ++n;
    }
    if (n > INT32_MAX) { c.err = "row total exceeds int32"; return CPH_E_INVALID; }
    row_ptr[k + 1] = (int32_t)n;
  }
  return CPH_OK;
}

static cph_status emit_pairs(std::vector<std::pair<int, int>> &out, int32_t *pairs, int64_t cap, int64_t *n) {
  std::sort(out.begin(), out.end());
  *n = (int64_t)out.size();
  if (pairs && cap >= (int64_t)out.size())
    for (size_t k = 0; k < out.size(); ++k) { pairs[2 * k] = out[k].first; pairs[2 * k + 1] = out[k].second; }
  return CPH_OK;
}

static cph_status sub_get_pairlist(SubCtx *ctx, int32_t r, int32_t *pairs, int64_t cap, int64_t *n) {
  CPH_NVTX("cph_get_pairlist");
  if (!ctx || !n) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  std::vector<std::pair<int, int>> all;
  if ((st = decode_directed(c, r, all))) return st;
  std::vector<std::pair<int, int>> out;
  for (auto &p : all)
    if (p.first < p.second) out.push_back(p);
  return emit_pairs(out, pairs, cap, n);
}

static cph_status sub_get_pairlist_directed(SubCtx *ctx, int32_t r, int32_t *pairs, int64_t cap, int64_t *n) {
  CPH_NVTX("cph_get_pairlist_directed");
  if (!ctx || !n) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  std::vector<std::pair<int, int>> all;
  if ((st = decode_directed(c, r, all))) return st;
  return emit_pairs(all, pairs, cap, n);
}

static cph_status sub_get_lambda_groups(SubCtx *ctx, int32_t r, int32_t *group_ptr, int32_t *coord_ptr, int32_t *atoms,
                                 int32_t *slot_atoms) {
  if (!ctx || !group_ptr || !coord_ptr || !atoms || !slot_atoms) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  const KParams &kp = c.kp;
  const size_t N = kp.N, base = (size_t)r * kp.Nst;
  std::vector<int> iperm(N);
  std::vector<int2> meta(N);
  CK(cudaMemcpy(iperm.data(), c.d.iperm + (size_t)r * N, sizeof(int) * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(meta.data(), c.d.meta + base, sizeof(int2) * N, cudaMemcpyDeviceToHost));
  if (kp.G) {
    CK(cudaMemcpy(group_ptr, c.d.g_ptr, sizeof(int) * (kp.G + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(coord_ptr, c.d.g_cptr, sizeof(int) * (kp.G + 1), cudaMemcpyDeviceToHost));
  } else {
    group_ptr[0] = coord_ptr[0] = 0;
  }
  std::vector<int> g_atoms(kp.nlam);
  if (kp.nlam) CK(cudaMemcpy(g_atoms.data(), c.d.g_atoms, sizeof(int) * kp.nlam, cudaMemcpyDeviceToHost));
  // device path 1: lambda slot k -> sorted slot (iperm of the stored atom) -> original index
  for (int k = 0; k < kp.nlam; ++k) atoms[k] = meta[iperm[g_atoms[k]]].x;
  // device path 2: the lambda slot each sorted slot's meta word carries -> original index
  for (int k = 0; k < kp.nlam; ++k) slot_atoms[k] = -1;
  for (size_t sl = 0; sl < N; ++sl) {
    const int ls = (meta[sl].y >> 8) - 1;
    if (ls >= 0 && ls < kp.nlam) slot_atoms[ls] = meta[sl].x;
  }
  return CPH_OK;
}

static cph_status sub_get_ti_means(SubCtx *ctx, int32_t r, double *mean, int64_t *n_samples) {
  if (!ctx) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  long long n = 0;
  CK(cudaMemcpy(&n, c.d.ti_n, sizeof(long long), cudaMemcpyDeviceToHost));
  std::vector<double> s(c.kp.C);
  if (c.kp.C) CK(cudaMemcpy(s.data(), c.d.ti_sum + (size_t)r * c.kp.C, sizeof(double) * c.kp.C, cudaMemcpyDeviceToHost));
  for (int k = 0; k < c.kp.C && mean; ++k) mean[k] = n ? s[k] / (double)n : 0.0;
  if (n_samples) *n_samples = n;
  return CPH_OK;
}

// blob: int64 magic, N, C, step | float pos[3N], vel[3N] | double lam[C], lamv[C]
static const int64_t kMagic = 0x3148504331ll;

static size_t state_bytes(const Ctx &c) {
  return 4 * sizeof(int64_t) + 6 * (size_t)c.kp.N * sizeof(float) + 2 * (size_t)c.kp.C * sizeof(double);
}

static cph_status ensure_state_buf(Ctx &c) {
  if (!c.h_bad) {
    CK(cudaMallocHost(&c.h_bad, 2 * sizeof(int)));
    c.h_bad[0] = c.h_bad[1] = 0;
  }
  if (c.d.state_buf) return CPH_OK;
  c.d.state_buf = dalloc<char>(c, state_bytes(c) * c.kp.R);
  if (!c.d.state_buf) { c.err = "device allocation failed"; return CPH_E_OOM; }
  return CPH_OK;
}

// replicas [r0, r0 + nr) -> host blobs (packed on the device, one copy), enqueued; the caller
// synchronises the stream before reading buf
static cph_status get_states_enqueue(Ctx &c, int r0, int nr, void *buf) {
  cph_status st = ensure_state_buf(c);
  if (st) return st;
  const size_t one = state_bytes(c);
  c.launches += launch_pack_state(c, c.stream, c.d.state_buf, (long long)one, r0, nr, c.host_step);
  CK(cudaMemcpyAsync(buf, c.d.state_buf, one * nr, cudaMemcpyDeviceToHost, c.stream));
  return CPH_OK;
}

static cph_status get_states(Ctx &c, int r0, int nr, void *buf) {
  cph_status st = get_states_enqueue(c, r0, nr, buf);
  if (st) return st;
  CK(cudaStreamSynchronize(c.stream));
  return CPH_OK;
}

// host blobs -> replicas [r0, r0 + nr), in three stages so that several sub-batches can run
// them side by side: (1) headers checked on the host, the blobs uploaded and checked for
// finiteness on the device (flag read back into pinned c.h_bad); (2) after a stream sync,
// reject a non-finite state before anything is overwritten; (3) unpack, move the clock, restart
// the TI accumulators and evaluate the new configuration (enqueued).
static cph_status set_states_begin(Ctx &c, int r0, int nr, const void *buf, int64_t nbytes, int64_t *step_out) {
  const size_t one = state_bytes(c);
  if (nbytes < (int64_t)(one * nr)) { c.err = "state blob too small"; return CPH_E_INVALID; }
  int64_t blob_step = -1;
  for (int k = 0; k < nr; ++k) {
    int64_t hdr[4];
    std::memcpy(hdr, (const char *)buf + one * k, sizeof hdr);
    if (hdr[0] != kMagic || hdr[1] != (int64_t)c.kp.N || hdr[2] != (int64_t)c.kp.C) {
      c.err = "state blob does not match this context";
      return CPH_E_INVALID;
    }
    if (hdr[3] < 0 || (k > 0 && hdr[3] != blob_step)) {
      c.err = "state blobs carry different (or negative) steps";
      return CPH_E_INVALID;
    }
    blob_step = hdr[3];
  }
  // The step is part of the state: the Philox noise is keyed on (seed, step) and frames,
  // nstlist/nstout phases and DBO blocks count from it, so a restore continues the run.  The
  // context has one clock: a full restore moves it, a partial one must match it.
  const bool all = r0 == 0 && nr == c.kp.R;
  if (!all && blob_step != c.host_step) {
    c.err = "state blob step differs from the context's step (restore every replica with cph_set_state_all "
            "to move the clock)";
    return CPH_E_STATE;
  }
  cph_status st = ensure_state_buf(c);
  if (st) return st;
  CK(cudaMemcpyAsync(c.d.state_buf, buf, one * nr, cudaMemcpyHostToDevice, c.stream));
  c.launches += launch_check_state(c, c.stream, c.d.state_buf, (long long)one, nr);
  CK(cudaMemcpyAsync(c.h_bad, c.d.flags + FLAG_BAD_STATE, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  *step_out = blob_step;
  return CPH_OK;
}

static cph_status set_states_rejected(Ctx &c) {
  if (!*c.h_bad) return CPH_OK;
  *c.h_bad = 0;
  const int zero = 0;
  CK(cudaMemcpy(c.d.flags + FLAG_BAD_STATE, &zero, sizeof(int), cudaMemcpyHostToDevice));
  c.err = "non-finite state";
  return CPH_E_INVALID;
}

static cph_status set_states_apply(Ctx &c, int r0, int nr, int64_t blob_step) {
  const size_t one = state_bytes(c);
  c.launches += launch_unpack_state(c, c.stream, c.d.state_buf, (long long)one, r0, nr);
  if (r0 == 0 && nr == c.kp.R && blob_step != c.host_step) {
    c.host_step = blob_step;
    k_set_end<<<1, 1, 0, c.stream>>>(c.d.step, blob_step);
    c.launches += 1;
  }
  // a new configuration: TI accumulators restart
  CK(cudaMemsetAsync(c.d.ti_sum, 0, sizeof(double) * (size_t)c.kp.R * c.kp.C, c.stream));
  CK(cudaMemsetAsync(c.d.ti_n, 0, sizeof(long long), c.stream));
  // re-sort and rebuild unless every restored atom sits where the last rebuild put it (a
  // restart of the configuration the list was built for, e.g. a checkpoint loop)
  CK(cudaMemsetAsync(c.d.flags + FLAG_MOVED, 0, sizeof(int), c.stream));
  c.launches += launch_list_moved(c, c.stream, r0, nr);
  CK(cudaMemcpyAsync(c.h_bad + 1, c.d.flags + FLAG_MOVED, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return evaluate_here(c, c.h_bad[1] != 0);
}

static cph_status set_states(Ctx &c, int r0, int nr, const void *buf, int64_t nbytes) {
  int64_t step = 0;
  cph_status st = set_states_begin(c, r0, nr, buf, nbytes, &step);
  if (st) return st;
  CK(cudaStreamSynchronize(c.stream));
  if ((st = set_states_rejected(c)) || (st = set_states_apply(c, r0, nr, step))) return st;
  // the re-evaluation is enqueued, not awaited: a device-side failure in it (list overflow,
  // divergence) is latched and reported by the next call, as for cph_step
  return CPH_OK;
}

static cph_status sub_get_state(SubCtx *ctx, int32_t r, void *buf, int64_t cap, int64_t *n) {
  CPH_NVTX("cph_get_state");
  if (!ctx || !n) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st) return st;
  *n = (int64_t)state_bytes(c);
  if (!buf) return CPH_OK;
  if (cap < *n) { c.err = "state buffer too small"; return CPH_E_INVALID; }
  cudaSetDevice(c.device);
  if ((st = sub_sync(ctx))) return st;
  return get_states(c, r, 1, buf);
}

static cph_status sub_set_state(SubCtx *ctx, int32_t r, const void *buf, int64_t nbytes) {
  CPH_NVTX("cph_set_state");
  if (!ctx || !buf) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cph_status st = check_replica(c, r);
  if (st || (st = sub_sync(ctx))) return st;
  return set_states(c, r, 1, buf, nbytes);
}

static cph_status sub_get_state_all(SubCtx *ctx, void *buf, int64_t cap, int64_t *n) {
  CPH_NVTX("cph_get_state_all");
  if (!ctx || !n) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  *n = (int64_t)(state_bytes(c) * c.kp.R);
  if (!buf) return CPH_OK;
  if (cap < *n) { c.err = "state buffer too small"; return CPH_E_INVALID; }
  cudaSetDevice(c.device);
  cph_status st = get_states_enqueue(c, 0, c.kp.R, buf);   // behind the queued work; flags checked after
  if (st) return st;
  return sub_sync(ctx);
}

static cph_status sub_set_state_all(SubCtx *ctx, const void *buf, int64_t nbytes) {
  CPH_NVTX("cph_set_state_all");
  if (!ctx || !buf) return CPH_E_INVALID;
  Ctx &c = ctx->c;
  cudaSetDevice(c.device);
  cph_status st = sub_sync(ctx);
  if (st) return st;
  return set_states(c, 0, c.kp.R, buf, nbytes);
}

// Eager steps of every sub-batch with CUDA events around each kernel class on `main`: per step
// and class, the sub-batches' launches of that class run concurrently on their own streams
// (fork from / join to `main`), so a class time is that of the kernel over the whole batch, as
// in the stepped graph, not of S smaller serialised launches.  Classes are serialised.
static cph_status profile_batches(const std::vector<Ctx *> &cs, const std::vector<cudaStream_t> &ss,
                                  cudaStream_t main, int64_t n_steps, double *ms, int64_t *launches) {
  Ctx &c = *cs[0];
  cudaSetDevice(c.device);
  const size_t S = cs.size();
  std::vector<cudaEvent_t> evs, joins(S, nullptr);
  std::vector<int> cls;
  cudaEvent_t fork = nullptr;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  for (auto &e : joins) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  static const char *kClassNames[] = {"integrate", "pairlist", "nonbonded", "spread", "fft_r2c", "solve",
                                      "fft_c2r", "gather", "lambda", "hi"};
  auto mark = [&](int k) {
    if (k >= 0 && k < (int)(sizeof(kClassNames) / sizeof(kClassNames[0]))) nvtxMarkA(kClassNames[k]);
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, main);
    evs.push_back(e);
    cls.push_back(k);
  };
  int64_t cnt[CPH_N_KCLASSES] = {0};
  // one kernel class over every sub-batch, concurrently; returns launches
  auto phase = [&](int k, auto &&fn) {
    cudaEventRecord(fork, main);
    for (size_t b = 0; b < S; ++b)
      if (ss[b] != main) cudaStreamWaitEvent(ss[b], fork, 0);
    int q = 0;
    for (size_t b = 0; b < S; ++b) q += fn(*cs[b], ss[b]);
    for (size_t b = 0; b < S; ++b)
      if (ss[b] != main) {
        cudaEventRecord(joins[b], ss[b]);
        cudaStreamWaitEvent(main, joins[b], 0);
      }
    if (k >= 0) cnt[k] += q;
    cs[0]->launches += q;
    mark(k);
  };
  const long long end = c.host_step + n_steps;
  mark(-1);
  phase(CPH_K_LAMBDA, [&](Ctx &x, cudaStream_t s) {
    k_set_end<<<1, 1, 0, s>>>(x.d.end_step, end);
    cufftSetStream(x.plan_r2c, s);
    cufftSetStream(x.plan_c2r, s);
    return 1 + launch_lambda_open(x, s);
  });
  cnt[CPH_K_LAMBDA] -= (int64_t)S;   // k_set_end is not a lambda kernel
  long long t = c.host_step;
  while (t < end) {
    const bool rebuild = (t + 1) % c.kp.nstlist == 0;
    phase(CPH_K_INTEGRATE, [&](Ctx &x, cudaStream_t s) { return launch_integrate(x, s, 1); });
    if (rebuild) phase(CPH_K_PAIRLIST, [&](Ctx &x, cudaStream_t s) { return launch_rebuild(x, s); });
    phase(CPH_K_NONBONDED, [&](Ctx &x, cudaStream_t s) { return launch_nonbonded(x, s, 1); });
    phase(CPH_K_SPREAD, [&](Ctx &x, cudaStream_t s) { return launch_spread(x, s); });
    phase(CPH_K_FFT_R2C, [&](Ctx &x, cudaStream_t) {
      fft_forward(x);
      return 0;
    });
    phase(CPH_K_SOLVE, [&](Ctx &x, cudaStream_t s) { return launch_solve(x, s, 1); });
    phase(CPH_K_FFT_C2R, [&](Ctx &x, cudaStream_t s) {
      fft_backward(x);
      return launch_grid_to32(x, s);
    });
    phase(CPH_K_GATHER, [&](Ctx &x, cudaStream_t s) { return launch_gather(x, s); });
    if (c.kp.hi)
      phase(CPH_K_HI, [&](Ctx &x, cudaStream_t s) { return launch_hi_recip(x, s) + launch_hi_finish(x, s, 1); });
    phase(CPH_K_LAMBDA, [&](Ctx &x, cudaStream_t s) { return launch_lambda_reduce(x, s, 1); });
    ++t;
  }
  phase(CPH_K_INTEGRATE, [&](Ctx &x, cudaStream_t s) { return launch_close(x, s, 1); });
  for (Ctx *x : cs) x->host_step = end;
  CK(cudaStreamSynchronize(main));
  double acc[CPH_N_KCLASSES] = {0};
  for (size_t e = 1; e < evs.size(); ++e) {
    float tm = 0.f;
    cudaEventElapsedTime(&tm, evs[e - 1], evs[e]);
    acc[cls[e]] += tm;
  }
  for (auto e : evs) cudaEventDestroy(e);
  for (auto e : joins) cudaEventDestroy(e);
  cudaEventDestroy(fork);
  if (ms) for (int q = 0; q < CPH_N_KCLASSES; ++q) ms[q] = acc[q];
  if (launches) for (int q = 0; q < CPH_N_KCLASSES; ++q) launches[q] = cnt[q];
  CK(cudaGetLastError());
  for (Ctx *x : cs)
    if (cph_status st = check_flags(*x)) {
      if (x != &c) c.err = x->err;
      return st;
    }
  return CPH_OK;
}

// ---- public API: a context = S replica sub-batches stepped concurrently ----------------------
// Each sub-batch is a complete single-batch context (SubCtx above) over a consecutive replica
// range with its own stream; with S > 1 the caller's stream forks into the sub-batch streams
// and joins back around every enqueuing call, so the public ordering contract (everything on
// cph_get_stream) is unchanged.  cph_step interleaves the sub-batches block by block: the
// PME chain of one batch (FFTs, solve, gather, lambda reduction: a few hundred CTAs at
// most) then overlaps the other batch's pair kernel instead of idling SMs at every step end
// (profiles/r02_summary.md).
struct cph_ctx {
  std::vector<SubCtx *> sub;
  std::vector<int> first;          // local replica index of each sub-batch's replica 0
  int R = 0, P = 0, remd_total = 0, nstlist = 1;
  int device = 0;
  cudaStream_t stream = nullptr;   // the public stream
  bool own_stream = false;
  std::vector<cudaStream_t> sstream;
  cudaEvent_t ev_in = nullptr;
  std::vector<cudaEvent_t> ev_out;
  double *rows = nullptr;          // cph_exchange scratch (S > 1; freed with batch 0)
  std::vector<cph_dbo_event> events;
  std::string err;
};

namespace {

cph_status fwd(cph_ctx *ctx, int s, cph_status st) {
  if (st != CPH_OK) ctx->err = ctx->sub[s]->c.err;
  return st;
}

// sub-batch holding local replica r, and its index there
int locate(cph_ctx *ctx, int r, int *rl) {
  if (r < 0 || r >= ctx->R) {
    ctx->err = "replica index out of range";
    return -1;
  }
  int s = (int)ctx->sub.size() - 1;
  while (ctx->first[s] > r) --s;
  *rl = r - ctx->first[s];
  return s;
}

// order the sub-batch streams after / before the public stream (no-ops for S = 1)
cph_status fork_in(cph_ctx *ctx) {
  if (ctx->sub.size() < 2) return CPH_OK;
  cudaSetDevice(ctx->device);
  if (cudaEventRecord(ctx->ev_in, ctx->stream) != cudaSuccess) { ctx->err = "cudaEventRecord failed"; return CPH_E_CUDA; }
  for (cudaStream_t s : ctx->sstream)
    if (cudaStreamWaitEvent(s, ctx->ev_in, 0) != cudaSuccess) { ctx->err = "cudaStreamWaitEvent failed"; return CPH_E_CUDA; }
  return CPH_OK;
}

cph_status join_out(cph_ctx *ctx) {
  if (ctx->sub.size() < 2) return CPH_OK;
  cudaSetDevice(ctx->device);
  for (size_t s = 0; s < ctx->sstream.size(); ++s)
    if (cudaEventRecord(ctx->ev_out[s], ctx->sstream[s]) != cudaSuccess ||
        cudaStreamWaitEvent(ctx->stream, ctx->ev_out[s], 0) != cudaSuccess) {
      ctx->err = "stream join failed";
      return CPH_E_CUDA;
    }
  return CPH_OK;
}

void destroy_composite(cph_ctx *ctx) {
  for (SubCtx *s : ctx->sub) sub_destroy(s);
  cudaSetDevice(ctx->device);
  for (cudaStream_t s : ctx->sstream) cudaStreamDestroy(s);
  for (cudaEvent_t e : ctx->ev_out) cudaEventDestroy(e);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int level_of(const cph_params *prm, double pH) {
  for (int p = 0; p < prm->n_ph_levels; ++p)
    if (std::fabs(pH - prm->ph_levels[p]) <= 1e-9 * std::max(1.0, std::fabs(prm->ph_levels[p]))) return p;
  return -1;
}

}  // namespace

extern "C" {

const char *cph_last_error(const cph_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

cph_status cph_create(const cph_system *sys, const cph_params *prm, cph_ctx **out) {
  CPH_NVTX("cph_create");
  if (!out) { g_create_err = "out is NULL"; return CPH_E_INVALID; }
  *out = nullptr;
  if (!sys || !prm) { g_create_err = "system/params is NULL"; return CPH_E_INVALID; }
  if (prm->abi_version != CPH_ABI_VERSION) { g_create_err = "abi_version mismatch"; return CPH_E_INVALID; }
  const int R = prm->n_replicas;
  if (R < 1) { g_create_err = "n_replicas must be >= 1"; return CPH_E_INVALID; }
  if (prm->sub_batches < 0) { g_create_err = "sub_batches must be >= 0"; return CPH_E_INVALID; }
  // automatic: up to 4 batches once the whole batch holds >= 24k atoms (measured on B200 over
  // C1..C5 x 2..64 replicas: 4 to 19 % less time per step; below that size the
  // step is launch-bound and extra batches only add launches)
  int S = prm->sub_batches ? prm->sub_batches : ((int64_t)R * sys->n_atoms >= 24000 ? 4 : 1);
  S = std::min(S, R);
  if (const char *e = getenv("CPH_SUB_BATCHES")) S = std::max(1, std::min(R, atoi(e)));   // A/B override
  // a ladder split across sub-batches is checked here (each sub-batch checks the ladders it
  // holds whole); a pH outside the levels is reported by the sub-batch
  if (S > 1 && prm->n_ph_levels >= 2 && prm->ph_levels && prm->pH) {
    std::vector<int> lab(R);
    bool all = true;
    for (int r = 0; r < R; ++r) all = all && (lab[r] = level_of(prm, prm->pH[r])) >= 0;
    if (all && !labels_form_ladders(lab.data(), R, prm->remd_first, prm->n_ph_levels)) {
      g_create_err = "each pH ladder held by this context must carry every level exactly once";
      return CPH_E_INVALID;
    }
  }
  cph_ctx *ctx = new cph_ctx;
  ctx->R = R;
  ctx->P = prm->n_ph_levels;
  ctx->remd_total = prm->remd_total ? prm->remd_total : R;
  ctx->nstlist = std::max(1, prm->nstlist);
  ctx->device = prm->device;
  auto fail = [&](cph_status st, const std::string &m) {
    g_create_err = m;
    destroy_composite(ctx);
    return st;
  };
  if (S == 1) {
    SubCtx *s0 = nullptr;
    cph_params p1 = *prm;
    p1.sub_batches = 1;
    cph_status st = sub_create(sys, &p1, &s0);
    if (st) { delete ctx; return st; }   // g_create_err set by sub_create
    ctx->sub.push_back(s0);
    ctx->first.push_back(0);
    ctx->stream = s0->c.stream;
    *out = ctx;
    return CPH_OK;
  }
  if (cudaSetDevice(prm->device) != cudaSuccess) return fail(CPH_E_CUDA, "cudaSetDevice failed");
  if (prm->cuda_stream) ctx->stream = (cudaStream_t)prm->cuda_stream;
  else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(CPH_E_CUDA, "stream creation failed");
    ctx->own_stream = true;
  }
  if (cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess)
    return fail(CPH_E_CUDA, "event creation failed");
  int C = 0, N = sys->n_atoms, off = 0;
  for (int s = 0; s < S; ++s) {
    const int Rs = R / S + (s < R % S ? 1 : 0);
    cudaStream_t st_s = nullptr;
    cudaEvent_t ev = nullptr;
    if (cudaStreamCreateWithFlags(&st_s, cudaStreamNonBlocking) != cudaSuccess)
      return fail(CPH_E_CUDA, "stream creation failed");
    ctx->sstream.push_back(st_s);
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      return fail(CPH_E_CUDA, "event creation failed");
    ctx->ev_out.push_back(ev);
    cph_params ps = *prm;
    ps.n_replicas = Rs;
    ps.sub_batches = 1;
    ps.cuda_stream = st_s;
    if (prm->pH) ps.pH = prm->pH + off;
    if (prm->replica_seed) ps.replica_seed = prm->replica_seed + off;
    if (prm->lambda0) ps.lambda0 = prm->lambda0 + (size_t)off * C;   // C known after batch 0 (off = 0 there)
    if (prm->pos_replicas) ps.pos_replicas = prm->pos_replicas + (size_t)off * N * 3;
    if (prm->vel_replicas) ps.vel_replicas = prm->vel_replicas + (size_t)off * N * 3;
    if (prm->n_ph_levels) {
      ps.remd_first = prm->remd_first + off;
      ps.remd_total = ctx->remd_total;
    }
    SubCtx *sc = nullptr;
    cph_status st = sub_create(sys, &ps, &sc);
    if (st) return fail(st, g_create_err);
    ctx->sub.push_back(sc);
    ctx->first.push_back(off);
    C = sc->c.kp.C;
    off += Rs;
  }
  if (ctx->P && ctx->remd_total == R) {   // cph_exchange scratch, owned by batch 0's allocations
    ctx->rows = dalloc<double>(ctx->sub[0]->c, (size_t)R * (ctx->P + 1));
    if (!ctx->rows) return fail(CPH_E_OOM, "device allocation failed");
  }
  // the sub-batches evaluated step 0 on their own streams: order the public stream after them
  if (join_out(ctx)) return fail(CPH_E_CUDA, ctx->err);
  *out = ctx;
  return CPH_OK;
}

void cph_destroy(cph_ctx *ctx) {
  if (!ctx) return;
  destroy_composite(ctx);
}

void *cph_get_stream(const cph_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }
int32_t cph_n_coords(const cph_ctx *ctx) { return ctx ? sub_n_coords(ctx->sub[0]) : -1; }
int32_t cph_n_atoms(const cph_ctx *ctx) { return ctx ? sub_n_atoms(ctx->sub[0]) : -1; }
int32_t cph_n_replicas(const cph_ctx *ctx) { return ctx ? ctx->R : -1; }
int32_t cph_n_sub_batches(const cph_ctx *ctx) { return ctx ? (int32_t)ctx->sub.size() : -1; }
int64_t cph_current_step(const cph_ctx *ctx) { return ctx ? sub_current_step(ctx->sub[0]) : -1; }
int64_t cph_launch_count(const cph_ctx *ctx) {
  if (!ctx) return -1;
  int64_t n = 0;
  for (SubCtx *s : ctx->sub) n += sub_launch_count(s);
  return n;
}

cph_status cph_step(cph_ctx *ctx, int64_t n_steps) {
  CPH_NVTX("cph_step");
  if (!ctx) return CPH_E_INVALID;
  if (n_steps < 0) { ctx->err = "n_steps < 0"; return CPH_E_INVALID; }
  if (n_steps == 0) return CPH_OK;
  if (ctx->sub.size() == 1) return fwd(ctx, 0, sub_step(ctx->sub[0], n_steps));
  cph_status st = fork_in(ctx);
  if (st) return st;
  // interleave the sub-batches in chunks of 32 nstlist blocks (aligned to the rebuild phase, so
  // full blocks replay the captured graphs): long enough that the per-segment cost (the
  // k_close / k_lambda_open pair and a graph launch that can no longer be pipelined behind
  // the previous one, ~0.1-0.3 ms measured) is rare, short enough that a long cph_step call
  // keeps every sub-batch stream fed instead of filling the launch queue with one of them
  static const long long chunk_blocks = getenv("CPH_SUB_CHUNK") ? atoll(getenv("CPH_SUB_CHUNK")) : 32;
  const long long chunk = chunk_blocks > 0 ? chunk_blocks * ctx->nstlist : n_steps;
  long long t = sub_current_step(ctx->sub[0]);
  const long long end = t + n_steps;
  while (t < end) {
    const long long next = std::min<long long>(end, (t / ctx->nstlist) * ctx->nstlist + chunk);
    for (size_t s = 0; s < ctx->sub.size(); ++s)
      if ((st = fwd(ctx, (int)s, sub_step(ctx->sub[s], next - t)))) return st;
    t = next;
  }
  return join_out(ctx);
}

cph_status cph_sync(cph_ctx *ctx) {
  CPH_NVTX("cph_sync");
  if (!ctx) return CPH_E_INVALID;
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if (cph_status st = fwd(ctx, (int)s, sub_sync(ctx->sub[s]))) return st;
  if (ctx->sub.size() > 1 && cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    ctx->err = "cudaStreamSynchronize failed";
    return CPH_E_CUDA;
  }
  return CPH_OK;
}

// per-replica calls: route to the sub-batch; enqueuing ones fork / join around the call
#define CPH_ROUTE(call_expr, enqueues)                                  \
  if (!ctx) return CPH_E_INVALID;                                     \
  int rl = 0;                                                         \
  const int s = locate(ctx, r, &rl);                                  \
  if (s < 0) return CPH_E_INVALID;                                    \
  SubCtx *sc = ctx->sub[s];                                           \
  if (enqueues) { if (cph_status e0 = fork_in(ctx)) return e0; }      \
  cph_status st_ = fwd(ctx, s, call_expr);                            \
  if (enqueues) { if (cph_status e1 = join_out(ctx)) return e1; }     \
  return st_;

cph_status cph_set_pH(cph_ctx *ctx, int32_t r, double pH) { CPH_ROUTE(sub_set_pH(sc, rl, pH), true) }
cph_status cph_get_lambdas(cph_ctx *ctx, int32_t r, double *lam, double *vel) {
  CPH_ROUTE(sub_get_lambdas(sc, rl, lam, vel), false)
}
cph_status cph_get_dvdl(cph_ctx *ctx, int32_t r, double *coul, double *bias) {
  CPH_ROUTE(sub_get_dvdl(sc, rl, coul, bias), false)
}
cph_status cph_get_bias_params(cph_ctx *ctx, int32_t r, double *d1) { CPH_ROUTE(sub_get_bias_params(sc, rl, d1), false) }
cph_status cph_get_energies(cph_ctx *ctx, int32_t r, double *e) { CPH_ROUTE(sub_get_energies(sc, rl, e), false) }
cph_status cph_get_frames_ex(cph_ctx *ctx, int32_t r, float *buf, uint8_t *censored, int64_t *steps, int32_t *labels,
                             int64_t cap, int64_t *n_frames, int64_t *n_dropped) {
  CPH_ROUTE(sub_get_frames_ex(sc, rl, buf, censored, steps, labels, cap, n_frames, n_dropped), false)
}
cph_status cph_get_frames(cph_ctx *ctx, int32_t r, float *buf, int64_t cap, int64_t *n_frames, int64_t *n_dropped) {
  CPH_ROUTE(sub_get_frames(sc, rl, buf, cap, n_frames, n_dropped), false)
}
cph_status cph_get_dbo_params(cph_ctx *ctx, int32_t r, double *p) { CPH_ROUTE(sub_get_dbo_params(sc, rl, p), false) }
cph_status cph_set_dbo_params(cph_ctx *ctx, int32_t r, const double *p) {
  CPH_ROUTE(sub_set_dbo_params(sc, rl, p), true)
}
cph_status cph_get_dbo_stats(cph_ctx *ctx, int32_t r, double *well, double *barrier) {
  CPH_ROUTE(sub_get_dbo_stats(sc, rl, well, barrier), false)
}
cph_status cph_get_forces(cph_ctx *ctx, int32_t r, float *f, float *phi) { CPH_ROUTE(sub_get_forces(sc, rl, f, phi), false) }
cph_status cph_get_positions(cph_ctx *ctx, int32_t r, float *pos, float *vel) {
  CPH_ROUTE(sub_get_positions(sc, rl, pos, vel), false)
}
cph_status cph_get_pairlist_rows(cph_ctx *ctx, int32_t r, const int32_t *atoms, int32_t n_atoms, int32_t *row_ptr,
                                 int32_t *cols, int64_t cap) {
  CPH_ROUTE(sub_get_pairlist_rows(sc, rl, atoms, n_atoms, row_ptr, cols, cap), false)
}
cph_status cph_get_pairlist(cph_ctx *ctx, int32_t r, int32_t *pairs, int64_t cap, int64_t *n) {
  CPH_ROUTE(sub_get_pairlist(sc, rl, pairs, cap, n), false)
}
cph_status cph_get_pairlist_directed(cph_ctx *ctx, int32_t r, int32_t *pairs, int64_t cap, int64_t *n) {
  CPH_ROUTE(sub_get_pairlist_directed(sc, rl, pairs, cap, n), false)
}
cph_status cph_get_lambda_groups(cph_ctx *ctx, int32_t r, int32_t *group_ptr, int32_t *coord_ptr, int32_t *atoms,
                                 int32_t *slot_atoms) {
  CPH_ROUTE(sub_get_lambda_groups(sc, rl, group_ptr, coord_ptr, atoms, slot_atoms), false)
}
cph_status cph_get_ti_means(cph_ctx *ctx, int32_t r, double *mean, int64_t *n_samples) {
  CPH_ROUTE(sub_get_ti_means(sc, rl, mean, n_samples), false)
}
cph_status cph_get_state(cph_ctx *ctx, int32_t r, void *buf, int64_t cap, int64_t *n) {
  CPH_ROUTE(sub_get_state(sc, rl, buf, cap, n), false)
}
cph_status cph_set_state(cph_ctx *ctx, int32_t r, const void *buf, int64_t nbytes) {
  CPH_ROUTE(sub_set_state(sc, rl, buf, nbytes), true)
}
#undef CPH_ROUTE

cph_status cph_exchange_energies(cph_ctx *ctx, double *rows) {
  if (!ctx || !rows) return CPH_E_INVALID;
  cph_status st = fork_in(ctx);
  if (st) return st;
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if ((st = fwd(ctx, (int)s, sub_exchange_energies(ctx->sub[s], rows + (size_t)ctx->first[s] * (ctx->P + 1)))))
      return st;
  return join_out(ctx);
}

cph_status cph_exchange_apply(cph_ctx *ctx, const double *rows_all, uint64_t seed, int64_t attempt) {
  if (!ctx) return CPH_E_INVALID;
  cph_status st = fork_in(ctx);
  if (st) return st;
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if ((st = fwd(ctx, (int)s, sub_exchange_apply(ctx->sub[s], rows_all, seed, attempt)))) return st;
  return join_out(ctx);
}

cph_status cph_exchange(cph_ctx *ctx, uint64_t seed, int64_t attempt) {
  if (!ctx) return CPH_E_INVALID;
  if (ctx->sub.size() == 1) return fwd(ctx, 0, sub_exchange(ctx->sub[0], seed, attempt));
  if (!ctx->P) { ctx->err = "replica exchange is off (n_ph_levels = 0)"; return CPH_E_STATE; }
  if (!ctx->rows) { ctx->err = "cph_exchange needs every replica in this context"; return CPH_E_STATE; }
  // energies of every sub-batch are joined into the public stream before any apply forks
  cph_status st = cph_exchange_energies(ctx, ctx->rows);
  return st ? st : cph_exchange_apply(ctx, ctx->rows, seed, attempt);
}

cph_status cph_get_labels(cph_ctx *ctx, int32_t *labels) {
  if (!ctx || !labels) return CPH_E_INVALID;
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if (cph_status st = fwd(ctx, (int)s, sub_get_labels(ctx->sub[s], labels + ctx->first[s]))) return st;
  return CPH_OK;
}

cph_status cph_set_labels(cph_ctx *ctx, const int32_t *labels) {
  if (!ctx || !labels) return CPH_E_INVALID;
  if (ctx->P && ctx->sub.size() > 1) {
    for (int r = 0; r < ctx->R; ++r)
      if (labels[r] < 0 || labels[r] >= ctx->P) { ctx->err = "label out of range"; return CPH_E_INVALID; }
    if (!labels_form_ladders(labels, ctx->R, ctx->sub[0]->c.kp.remd_first, ctx->P)) {
      ctx->err = "each pH ladder held by this context must carry every level exactly once";
      return CPH_E_INVALID;
    }
  }
  cph_status st = fork_in(ctx);
  if (st) return st;
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if ((st = fwd(ctx, (int)s, sub_set_labels(ctx->sub[s], labels + ctx->first[s])))) return st;
  return join_out(ctx);
}

cph_status cph_get_exchange_stats(cph_ctx *ctx, int64_t *attempts, int64_t *accepts) {
  if (!ctx) return CPH_E_INVALID;
  // every sub-batch applies every ladder's decisions and counts them: batch 0's tally is the one
  for (size_t s = 1; s < ctx->sub.size(); ++s)
    if (cph_status st = fwd(ctx, (int)s, sub_sync(ctx->sub[s]))) return st;
  return fwd(ctx, 0, sub_get_exchange_stats(ctx->sub[0], attempts, accepts));
}

cph_status cph_get_dbo_events(cph_ctx *ctx, cph_dbo_event *ev, int64_t cap, int64_t *n) {
  if (!ctx || cap < 0 || (cap > 0 && !ev)) return CPH_E_INVALID;
  // drain every sub-batch, map to local replica indices, merge in (step, replica) order
  bool added = false;
  for (size_t s = 0; s < ctx->sub.size(); ++s) {
    std::vector<cph_dbo_event> &q = ctx->sub[s]->c.events;
    for (cph_dbo_event e : q) {
      e.replica += ctx->first[s];
      ctx->events.push_back(e);
      added = true;
    }
    q.clear();
  }
  if (added)
    std::stable_sort(ctx->events.begin(), ctx->events.end(), [](const cph_dbo_event &a, const cph_dbo_event &b) {
      return a.step != b.step ? a.step < b.step : a.replica < b.replica;
    });
  const int64_t take = std::min<int64_t>(cap, (int64_t)ctx->events.size());
  std::copy(ctx->events.begin(), ctx->events.begin() + take, ev);
  ctx->events.erase(ctx->events.begin(), ctx->events.begin() + take);
  if (n) *n = take;
  return CPH_OK;
}

cph_status cph_get_state_all(cph_ctx *ctx, void *buf, int64_t cap, int64_t *n) {
  CPH_NVTX("cph_get_state_all");
  if (!ctx || !n) return CPH_E_INVALID;
  if (ctx->sub.size() == 1) return fwd(ctx, 0, sub_get_state_all(ctx->sub[0], buf, cap, n));
  const int64_t one = (int64_t)state_bytes(ctx->sub[0]->c);
  *n = one * ctx->R;
  if (!buf) return CPH_OK;
  if (cap < *n) { ctx->err = "state buffer too small"; return CPH_E_INVALID; }
  cudaSetDevice(ctx->device);
  // every sub-batch packs and copies out behind its queued work, side by side (a batch's copy
  // overlaps the others' compute); latched device failures are checked once all have landed
  for (size_t s = 0; s < ctx->sub.size(); ++s) {
    Ctx &c = ctx->sub[s]->c;
    if (cph_status st = fwd(ctx, (int)s, get_states_enqueue(c, 0, c.kp.R, (char *)buf + one * ctx->first[s])))
      return st;
  }
  for (size_t s = 0; s < ctx->sub.size(); ++s)
    if (cph_status st = fwd(ctx, (int)s, sub_sync(ctx->sub[s]))) return st;
  return CPH_OK;
}

cph_status cph_set_state_all(cph_ctx *ctx, const void *buf, int64_t nbytes) {
  CPH_NVTX("cph_set_state_all");
  if (!ctx || !buf) return CPH_E_INVALID;
  if (ctx->sub.size() == 1) return fwd(ctx, 0, sub_set_state_all(ctx->sub[0], buf, nbytes));
  const size_t S = ctx->sub.size();
  const int64_t one = (int64_t)state_bytes(ctx->sub[0]->c);
  if (nbytes < one * ctx->R) { ctx->err = "state blob too small"; return CPH_E_INVALID; }
  cudaSetDevice(ctx->device);
  // every header is checked (all blobs one step) before any sub-batch is touched
  const Ctx &c0 = ctx->sub[0]->c;
  int64_t step0 = -1;
  for (int r = 0; r < ctx->R; ++r) {
    int64_t hdr[4];
    std::memcpy(hdr, (const char *)buf + one * r, sizeof hdr);
    if (hdr[0] != kMagic || hdr[1] != (int64_t)c0.kp.N || hdr[2] != (int64_t)c0.kp.C) {
      ctx->err = "state blob does not match this context";
      return CPH_E_INVALID;
    }
    if (hdr[3] < 0 || (r > 0 && hdr[3] != step0)) {
      ctx->err = "state blobs carry different (or negative) steps";
      return CPH_E_INVALID;
    }
    step0 = hdr[3];
  }
  cph_status st;
  for (size_t s = 0; s < S; ++s)
    if ((st = fwd(ctx, (int)s, sub_sync(ctx->sub[s])))) return st;
  if ((st = fork_in(ctx))) return st;
  // upload + finiteness check on every sub-batch; nothing is overwritten unless all pass
  std::vector<int64_t> steps(S);
  for (size_t s = 0; s < S; ++s) {
    Ctx &c = ctx->sub[s]->c;
    if ((st = fwd(ctx, (int)s, set_states_begin(c, 0, c.kp.R, (const char *)buf + one * ctx->first[s],
                                                 one * c.kp.R, &steps[s]))))
      return st;
  }
  cph_status rejected = CPH_OK;
  for (size_t s = 0; s < S; ++s) {
    Ctx &c = ctx->sub[s]->c;
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) { ctx->err = "cudaStreamSynchronize failed"; return CPH_E_CUDA; }
    if (cph_status r = set_states_rejected(c)) { if (!rejected) { rejected = r; ctx->err = c.err; } }
  }
  if (rejected) return rejected;
  for (size_t s = 0; s < S; ++s) {
    Ctx &c = ctx->sub[s]->c;
    if ((st = fwd(ctx, (int)s, set_states_apply(c, 0, c.kp.R, steps[s])))) return st;
  }
  // re-evaluations enqueued on every sub-batch; their device-side flags are checked by the next call
  return join_out(ctx);
}

cph_status cph_profile_steps(cph_ctx *ctx, int64_t n_steps, double *ms, int64_t *launches) {
  CPH_NVTX("cph_profile_steps");
  if (!ctx || n_steps < 0) return CPH_E_INVALID;
  std::vector<Ctx *> cs;
  std::vector<cudaStream_t> ss;
  for (SubCtx *s : ctx->sub) {
    cs.push_back(&s->c);
    ss.push_back(s->c.stream);
  }
  cph_status st = fork_in(ctx);
  if (st) return st;
  if ((st = fwd(ctx, 0, profile_batches(cs, ss, ctx->stream, n_steps, ms, launches)))) return st;
  return join_out(ctx);
}

}  // extern "C"
