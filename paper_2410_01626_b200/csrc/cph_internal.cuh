// Internal declarations of the cph library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/cph.h"

namespace cph {

// ---- physical constants (own copy; the oracle keeps its own) -----------------------
constexpr double kFCoul = 138.935458;        // kJ mol^-1 nm e^-2
constexpr double kBoltz = 0.0083144626;      // kJ mol^-1 K^-1
constexpr double kPi = 3.14159265358979323846;
constexpr double kLn10 = 2.30258509299404568402;

constexpr int kNE = CPH_N_ETERMS;
constexpr int kMaxTypes = 32;                // LJ table kept in shared memory

// neighbour-list entry: sorted slot j (21 bits) | LJ type of j (5 bits) | image code (5 bits)
// image code = (kx+1)*9 + (ky+1)*3 + (kz+1), k = rint((x_j - x_i)/L) at the rebuild
constexpr uint32_t kEntryJMask = 0x1FFFFFu;
constexpr int kEntryTypeShift = 21;
constexpr uint32_t kEntryTypeMask = 0x1Fu;
constexpr int kEntryImgShift = 26;
// padding entries (a lane's last tile, and the tiles past its count) name the atom itself with
// image code 0, i.e. shifted by a whole box diagonal: r^2 = |L|^2 > r_c^2, so the pair kernel's
// cutoff test alone discards them
constexpr uint32_t kPadCode = 0u;
constexpr int kMaxAtoms = 1 << 21;

// Device-side flags (int array)
enum { FLAG_PENDING_CLOSE = 0, FLAG_LIST_OVERFLOW = 1, FLAG_DIVERGED = 2, FLAG_MAX_NNB = 3,
       FLAG_STEP_DONE = 4, FLAG_BAD_STATE = 5, FLAG_REMD_BAD = 6, FLAG_MOVED = 7,
       FLAG_CL_OVERFLOW = 8, FLAG_CL_MAX = 9, FLAG_COUNT = 10 };

// cluster pair-list entry word: j-cluster index J (slots 4J..4J+3) | image code << kEntryImgShift
constexpr uint32_t kClJMask = 0x7FFFFu;
constexpr int kClI = 8;                      // atoms per i-cluster
constexpr int kClJ = 4;                      // atoms per j-cluster
constexpr int kClSuper = 32;                 // atoms per super-cluster (4 i-clusters, one warp)

// Scalars every kernel needs, passed by value.
struct KParams {
  int R, N, Nst;               // replicas, atoms, per-replica stride (multiple of 32)
  float L[3], invL[3];         // box (fp32) and 1/L (fp32, computed as 1.0f/L)
  double Ld[3];
  float rc2, rlist2;
  float beta, beta_p;          // Ewald beta, beta * p (erfc polynomial scale)
  float two_beta_sqrtpi;       // 2 beta / sqrt(pi)
  float fcoul;
  int T;                       // LJ types
  // cells
  int nc[3], ncell;            // cells per dimension, total
  int ns[3], so[3];            // stencil sizes and first offsets per dimension
  int nb_packed;               // pair kernel: FFMA2 path for non-lambda warps (A/B: CPH_NB_PACKED=0)
  int det;                     // deterministic (fixed-point) PME spread
  int fft64;                   // small grids (K^3 <= 32768): PME grid, FFTs and solve in fp64
  // list
  int cap;                     // neighbour capacity per atom (per-atom list; lambda-atom lists)
  int pair_mode;               // 0 per-atom full list, 1 cluster-pair list (cph_params.pair_list)
  int nsc;                     // super-cluster ids per replica (cluster mode): Nst/32 + columns + 1
  int clcap;                   // entries per super-cluster (cluster mode)
  // PME
  int K[3], K3, Kc;            // grid, K^3, complex points per replica
  int Kzc;                     // Kz/2+1
  float V;                     // volume nm^3
  // dynamics
  float dt, kT_f;
  double dtd, kT;
  float c1_atom, c2_atom_kT;   // exp(-g dt), (1-c1^2) kT
  double c1_lam, sd_lam;       // exp(-g_l dt), sqrt((1-c1^2) kT / m_l)
  double m_lam;
  int nstout, nstenergy, nstlist;
  int mode;
  // lambda groups
  int G, C, nlam;
  double beta_d;
  double Q_fixed, Q2_fixed;    // sum and sum of squares of fixed charges (per replica identical)
  double h_barrier, wall_k;
  int fcap;                    // frame capacity
  // DBO statistics: on/off and the proximity / transition bands
  int dbo_on;
  double dbo_near, dbo_trans_lo, dbo_trans_hi;
  // Bussi thermostat (R27/R28): on/off, degrees of freedom, exp(-dt/tau)
  int bussi;
  double nf_atom, cb_atom, cb_lam;
  // pH replica exchange (R29/R30): P levels (0 = off), global replica layout
  int P, remd_total, remd_first;
  // Hamiltonian interpolation (R31): on/off, reciprocal m-list size, table extents
  int hi, hi_nm, hi_kmax[3], hi_nsplit;
};

struct DevBufs {
  float4 *xyzq = nullptr, *xyzq_alt = nullptr;
  float4 *vel = nullptr, *vel_alt = nullptr;
  int2 *meta = nullptr, *meta_alt = nullptr;       // (orig, type | (lslot+1) << 8)
  float4 *f_nb = nullptr, *f_rec = nullptr;
  int *iperm = nullptr;                             // [R*N] orig -> slot
  int *cell_of = nullptr, *cell_rank = nullptr;     // [R*Nst]
  int *cell_count = nullptr, *cell_start = nullptr; // [R*ncell], [R*(ncell+1)]
  int *perm_tmp = nullptr;                          // [R*Nst] new slot -> old slot
  uint32_t *nbl = nullptr;                          // [R*cap*Nst]
  // cluster-pair list (pair_mode 1): per super-cluster id its first slot, atom count, entries
  uint32_t *cl_j = nullptr;                         // [R*nsc*clcap] J | image code << 26
  uint4 *cl_m = nullptr;                            // [R*nsc*clcap] interaction mask per i-cluster
  int *cl_n = nullptr, *sc_first = nullptr, *sc_ni = nullptr;   // [R*nsc]
  uint32_t *lam_nbl = nullptr;                      // [R*nlam*cap] full rows of the lambda atoms (slot | code << 26)
  int *lam_n = nullptr;                             // [R*nlam]
  int *nnb = nullptr;                               // [R*Nst]
  int *excl_ptr = nullptr, *excl_idx = nullptr;     // CSR by original atom
  float2 *ljtab = nullptr;                          // [T*T] (6 c6, 12 c12) fp32
  double *phi64_nb = nullptr;                       // [R*nlam]
  float *grid = nullptr;                            // [R*K3]
  float2 *cgrid = nullptr;                          // [R*Kc]
  float *bsp = nullptr;                             // [Kx + Ky + Kz] |b|^2 moduli
  float *ginf = nullptr;                            // [Kc] influence function G(m) (replica independent)
  double *grid64 = nullptr;                         // [R*K3] fp64 grid (fft64 mode)
  double2 *cgrid64 = nullptr;                       // [R*Kc] fp64 half spectrum (fft64 mode)
  double *ginf64 = nullptr;                         // [Kc] fp64 G(m) (fft64 mode)
  unsigned long long *grid_fx = nullptr;            // [R*K3] fixed-point spread accumulator (deterministic mode)
  int *g_kind = nullptr, *g_ptr = nullptr, *g_atoms = nullptr, *g_cptr = nullptr;
  double *g_q = nullptr;                            // [nlam*4]
  double *vmm = nullptr;                            // [G*36]
  double *g_dG = nullptr;                           // [R*G*3] dG macro, delta, eps at pH
  double *d1 = nullptr;                             // [R*C]
  double *lam = nullptr, *lamv = nullptr;           // [R*C]
  double *qlam = nullptr;                           // [R*nlam]
  double *dvdl_coul = nullptr, *dvdl_bias = nullptr;// [R*C]
  double *ti_sum = nullptr;                         // [R*C]
  long long *ti_n = nullptr;                        // [1]
  double *erec = nullptr;                           // [2*R*kNE]
  float *frames = nullptr;                          // [R*fcap*C]
  long long *frame_total = nullptr;                 // [R]
  long long *step = nullptr, *end_step = nullptr;   // device step counter, last step of call
  int *done_counter = nullptr;
  int *flags = nullptr;
  uint64_t *seed = nullptr;                         // [R]
  double *phi_lam = nullptr;                        // [R*nlam] total phi of lambda atoms
  int *k_group = nullptr;                           // [nlam] group of each lambda atom
  // DBO
  double *dw = nullptr;                             // [R*C*4] a0, a1, h_prot, h_deprot
  double *dbo_well = nullptr;                       // [R*C*5] block accumulators (well)
  double *dbo_bar = nullptr;                        // [R*C*4] block accumulators (barrier)
  int *c_group = nullptr;                           // [C] group of each coordinate
  int *c_lp = nullptr;                              // [C] lambda_p coordinate of a tautomer coordinate, else -1
  long long *cens = nullptr;                        // [R*G*2] censor window (from, until]
  unsigned char *frame_cens = nullptr;              // [R*fcap*C]
  long long *frame_step = nullptr;                  // [R*fcap]
  double *bussi_k = nullptr;                        // [2*R] mid-step atom kinetic energy by step parity
  // pH replica exchange
  double *lvl_d1 = nullptr;                         // [P*C] PFC depths per pH level
  double *lvl_dG = nullptr;                         // [P*G*3] dG per pH level
  int *remd_label = nullptr;                        // [R] level index of each local replica
  double *remd_rows = nullptr;                      // [R*(P+1)] (label, E_p) rows for cph_exchange
  int *remd_holder = nullptr, *remd_newlab = nullptr;   // [remd_total] scratch of the apply kernel
  long long *remd_att = nullptr, *remd_acc = nullptr;   // [L*(P-1)] attempts / accepts per pair
  int *frame_label = nullptr;                       // [R*fcap]
  // Hamiltonian interpolation
  int4 *hi_m = nullptr;                             // [hi_nm] half-space m (integers)
  float *hi_w = nullptr;                            // [hi_nm] 2 exp(-pi^2 m^2/beta^2)/(pi V m^2)
  uint32_t *hi_excl = nullptr;                      // [nlam] intra-group exclusion mask per atom
  double *hi_M = nullptr;                           // [R*G*10] reciprocal form matrix (without f)
  float *hi_F = nullptr;                            // [R*nlam*3] reciprocal force sums (without 4 pi f)
  char *state_buf = nullptr;                        // [R * state blob bytes] staging of get/set_state
  double *hi_dvdl = nullptr;                        // [R*C] dC/dlambda
};

struct DboConfig {
  int well = 0, barrier = 0;
  long long well_steps = 20000, barrier_steps = 500000, censor_steps = 5000;
  double near = 0.2, residency = 0.7, tol = 0.03, gain = 0.5, cap = 0.08;
  double trans_lo = 0.2, trans_hi = 0.8, target = 0.25, target_tol = 0.05;
  double bstep = 1.0, bmin = 1.0, bmax = 20.0;
};

struct Timeline {   // CPH_TIMELINE diagnostic (host.cu): %globaltimer stamps from 1-thread kernels
  static constexpr int S = 64, T = 12;
  int s = 0, n = 0;
  unsigned long long *stamps = nullptr;   // device [S][T]
  bool used[S][T] = {};
  double sum[S][T] = {};
};
struct Ctx {
  Timeline *tl = nullptr;                           // CPH_TIMELINE diagnostic (host.cu)
  KParams kp{};
  DevBufs d;
  cudaStream_t stream = nullptr, stream_pme = nullptr, stream_nb = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork2 = nullptr, ev_join2 = nullptr, ev_gather = nullptr;
  bool prio = false;                                // pair kernel on a high-priority stream
  bool own_stream = false;
  cufftHandle plan_r2c = 0, plan_c2r = 0;
  void *(*dev_alloc)(size_t, void *) = nullptr;
  void (*dev_free)(void *, void *) = nullptr;
  void *alloc_ctx = nullptr;
  std::vector<void *> allocations;
  int device = 0;
  // host copies
  std::vector<int> h_group_kind, h_group_ptr, h_group_atoms, h_cptr;
  std::vector<double> h_state_q, h_pKa, h_pH;
  std::vector<int> h_excl_ptr, h_excl_idx;
  std::vector<uint64_t> h_seed;
  std::vector<double> h_d1;                         // [R*C]
  std::vector<double> h_dG;                         // [R*G*3]
  std::vector<double> h_dw;                         // [R*C*4] DBO parameters (host master copy)
  std::vector<int> h_c_group, h_c_lp;               // [C]
  std::vector<long long> h_cens;                    // [R*G*2]
  std::vector<cph_dbo_event> events;                // undrained DBO log
  int *h_bad = nullptr;                             // pinned [2]: FLAG_BAD_STATE, FLAG_MOVED read back by set_state
  std::vector<double> h_levels;                     // [P] pH ladder
  std::vector<double> h_lvl_d1, h_lvl_dG;           // [P*C], [P*G*3]
  DboConfig dbo;
  int *h_flags_mapped = nullptr;                    // host view of a mapped flag copy
  int *d_flags_mapped = nullptr;
  long long host_step = 0;
  int64_t launches = 0;
  // CUDA graph of one nstlist block (rebuild at first step)
  cudaGraphExec_t graph_block = nullptr;
  int graph_block_kernels = 0;
  std::string err;
  size_t cap_grow = 0;
  size_t clcap_grow = 0;
};

// ---- launchers (each returns the number of kernels it launched) ----------------------
int launch_integrate(Ctx &c, cudaStream_t s, int do_open);       // BAOA (+ pending close); Bussi: BA + T A
int launch_close(Ctx &c, cudaStream_t s, int kick);                // final half kick / KE
int launch_rebuild(Ctx &c, cudaStream_t s);                        // sort + pair list
int launch_sort(Ctx &c, cudaStream_t s);                           // cell sort + permutation
int launch_build_list(Ctx &c, cudaStream_t s);                     // pair list of the sorted atoms
int launch_nonbonded(Ctx &c, cudaStream_t s, int step_offset);
int launch_spread(Ctx &c, cudaStream_t s);
int launch_solve(Ctx &c, cudaStream_t s, int step_offset);
int launch_influence(Ctx &c, cudaStream_t s);                      // G(m) table, once at create
int launch_gather(Ctx &c, cudaStream_t s);
int launch_grid_to32(Ctx &c, cudaStream_t s);                      // fft64 mode: grid64 -> grid after the back transform
int launch_lambda_reduce(Ctx &c, cudaStream_t s, int mode);       // 0 init eval, 1 step
int launch_lambda_open(Ctx &c, cudaStream_t s);
int launch_set_charges(Ctx &c, cudaStream_t s);
int launch_remd_energy(Ctx &c, cudaStream_t s, double *rows);
int launch_remd_apply(Ctx &c, cudaStream_t s, const double *rows_all, uint64_t seed, long long attempt);
int launch_bias_refresh(Ctx &c, cudaStream_t s);
int launch_hi_recip(Ctx &c, cudaStream_t s);
int launch_hi_finish(Ctx &c, cudaStream_t s, int step_offset);
// state blobs (original atom order) packed / checked / unpacked on the device
int launch_pack_state(Ctx &c, cudaStream_t s, char *dst, long long one, int r0, int nr, long long step);
int launch_check_state(Ctx &c, cudaStream_t s, const char *src, long long one, int nr);
int launch_unpack_state(Ctx &c, cudaStream_t s, const char *src, long long one, int r0, int nr);
int launch_list_moved(Ctx &c, cudaStream_t s, int r0, int nr);

// host PFC (pfc.cu); dw = (a0, a1, h_prot, h_deprot) of each coordinate of the site
bool pfc_two_state(const double dw[4], double pKa, double pH, double T, double kw, double *d1, std::string *err);
bool pfc_three_state(const double dwp[4], const double dwt[4], const double pKa3[3], double pH, double T,
                     double kw, double *d1p, double *d1t, std::string *err);
double delta_g(double pKa, double pH, double T);

}  // namespace cph
