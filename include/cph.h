/*
 * cph.h — C ABI of the B200 (sm_100a) constant-pH lambda-dynamics step library.
 *
 * What one step computes (arXiv 2410.01626 as read in DESIGN.md):
 *   a1  lambda -> charges, q_i = sum_s w_s(lp, lt) q_i^s with the Eq. 2 weights
 *       (PAPER.md:618-632); only charges differ between forms;
 *       charge-buffer oxygens switch -0.834 -> +0.166 e.
 *   a2  cell-list Verlet pair list, rebuilt every nstlist steps.
 *   a3  real-space Ewald + Lennard-Jones pair kernel accumulating forces and the
 *       per-atom potential phi_i.
 *   a4-a7  smooth PME: B-spline spread, 3D FFT (cuFFT), influence-function
 *       solve, potential/force gather.
 *   a8  dV/dlambda_k = f sum_{i in k} (dq_i/dlambda_k) phi_i reduced in fp64 per
 *       lambda-group, plus the bias V = Vmm + VpH + Vdw (Eq. 3, PAPER.md:667-698,
 *       :715-740).
 *   a9  BAOAB Langevin / velocity-Verlet update of atoms and lambda particles
 *       (m_lambda = 60 u), dt = 2 fs, 300 K;
 *   f2  or, instead of the Langevin O step, the paper's Bussi thermostat.
 *   f3  pH replica exchange across replicas / GPUs (cph_exchange*).
 *   f4  optional Hamiltonian interpolation (params.hamiltonian).
 *   a10 Partition Function Correction of the double-well depths at cph_create /
 *       cph_set_pH.
 *   f1  optional Dynamic Barrier and Well Optimization with censoring
 *       (R23-R26): per-step block statistics on the
 *       device, controller rules and PFC refresh on the host at block ends.
 *
 * Conventions
 *   Units: nm, ps, u, kJ/mol, e, K.  lambda = 0 is protonated; a frame is
 *   deprotonated iff lambda_p >= 0.5 (reading R1).
 *   Coordinates: group g of kind 2 owns one coordinate (lp); kind 3 (His-like)
 *   owns two (lp, lt).  The flat lambda vector of a replica concatenates them
 *   in group order; C = number of coordinates.
 *   Atom order: every getter returns ORIGINAL atom order (the order of
 *   cph_system.pos), whatever order the device keeps internally.
 *   Replicas: one context batches R replicas of the same system (same
 *   topology and box), which differ in pH, seed, initial lambda, positions and
 *   velocities.  Every kernel launch covers all R replicas.
 *
 * Ownership: input pointers are borrowed for the duration of the call and
 *   copied.  Output buffers are caller-owned host memory.  Device memory is
 *   owned by the context; it is obtained through params.dev_alloc/dev_free when
 *   given (the Python binding passes PyTorch's caching allocator) or cudaMalloc.
 * Errors: every call returns a cph_status; nothing throws across the ABI.
 *   cph_last_error(ctx) gives a message (ctx == NULL: last cph_create failure
 *   of this thread).  cph_step is asynchronous on params.cuda_stream; device
 *   side failures (lambda divergence |lambda| > 10 or non-finite dV/dlambda,
 *   pair-list overflow) are latched and reported by the next call.
 * Threading: a context is not thread-safe; use one per host thread.
 */
#ifndef CPH_H
#define CPH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPH_ABI_VERSION 5

typedef struct cph_ctx cph_ctx;

typedef enum {
  CPH_OK = 0,
  CPH_E_INVALID = 1,     /* invalid argument or inconsistent system */
  CPH_E_CUDA = 2,        /* CUDA / cuFFT runtime error */
  CPH_E_DIVERGED = 3,    /* |lambda| > 10 or non-finite dV/dlambda */
  CPH_E_STATE = 4,       /* call not valid in the current state (e.g. list overflow, rebuilt) */
  CPH_E_OOM = 5,         /* device allocation failed */
  CPH_E_UNSUPPORTED = 6  /* valid request outside what this build implements */
} cph_status;

/* energy terms returned by cph_get_energies, kJ/mol */
enum {
  CPH_E_LJ = 0, CPH_E_REAL, CPH_E_EXCL, CPH_E_SELF, CPH_E_RECIP, CPH_E_NET,
  CPH_E_HI,      /* Hamiltonian-interpolation correction sum_g C_g (0 unless params.hamiltonian) */
  CPH_E_BIAS, CPH_E_KE_ATOMS, CPH_E_KE_LAMBDA, CPH_E_TOTAL, CPH_N_ETERMS
};

/* kernel classes timed by cph_profile_steps */
enum {
  CPH_K_INTEGRATE = 0, CPH_K_PAIRLIST, CPH_K_NONBONDED, CPH_K_SPREAD, CPH_K_FFT_R2C,
  CPH_K_SOLVE, CPH_K_FFT_C2R, CPH_K_GATHER, CPH_K_LAMBDA, CPH_K_HI, CPH_N_KCLASSES
};

typedef struct {
  int32_t n_atoms;              /* N >= 1, N <= 2^21 */
  const float *pos;             /* [N*3] nm, any image */
  const float *vel;             /* [N*3] nm/ps or NULL (zero) */
  const float *mass;            /* [N] u; 0 = frozen (never moved) */
  const float *charge;          /* [N] e; used for atoms that are in no lambda-group */
  const int32_t *type;          /* [N] LJ type in [0, n_types) */
  int32_t n_types;              /* 1..255 */
  const double *c6;             /* [T*T] kJ mol^-1 nm^6, symmetric */
  const double *c12;            /* [T*T] kJ mol^-1 nm^12, symmetric */
  int32_t n_excl;               /* number of excluded pairs */
  const int32_t *excl;          /* [2*n_excl] unordered atom pairs, i != j */
  double box[3];                /* rectangular box edges, nm; the device simulates fl32(box) (R34) */
  int32_t n_groups;             /* G >= 0 lambda-groups */
  const int32_t *group_kind;    /* [G] 2 (one coordinate) or 3 (two coordinates) */
  const int32_t *group_ptr;     /* [G+1] CSR offsets into group_atoms */
  const int32_t *group_atoms;   /* [n_group_atoms] atom indices, each atom in <= 1 group */
  const double *state_q;        /* [n_group_atoms*4] charges of forms A,B,C,D (Eq. 2);
                                   kind 2 requires A == B and C == D */
  const int32_t *is_buffer;     /* [n_group_atoms] 1 for the charge-buffer member, or NULL */
  const double *pKa;            /* [G*3] macro, micro-delta, micro-eps (kind 2 uses macro) */
  const double *vmm;            /* [G*36] Vmm coefficients c[a*6+b] of lp^a lt^b */
} cph_system;

typedef struct {
  int32_t abi_version;          /* = CPH_ABI_VERSION */
  int32_t n_replicas;           /* R >= 1 */
  int32_t device;               /* CUDA device ordinal */
  int32_t mode;                 /* 0 lambda dynamics; 1 fixed-lambda TI (lambda frozen,
                                   dV/dlambda accumulated for cph_get_ti_means) */
  double dt;                    /* ps (0.002) */
  double temperature;           /* K (300) */
  double gamma_atom;            /* ps^-1 Langevin friction of atoms (1) */
  double gamma_lambda;          /* ps^-1 friction of lambda particles (1 = 1/tau) */
  double lambda_mass;           /* u (60) */
  double rc;                    /* nm real-space / LJ cut-off (1.0) */
  double rlist;                 /* nm pair-list radius (1.1), rc <= rlist < min(box)/2 */
  double ewald_rtol;            /* erfc(beta rc) = ewald_rtol (1e-5) */
  int32_t pme_grid[3];          /* K_x, K_y, K_z: even, factors 2,3,5,7 only */
  int32_t pme_order;            /* 4 (only order supported) */
  int32_t nstlist;              /* pair-list rebuild interval (10) */
  int32_t nstout;               /* lambda frame interval (250 = 0.5 ps) */
  int32_t nstenergy;            /* energy evaluation interval (250) */
  double barrier;               /* kJ/mol double-well barrier h (6) */
  double wall_k;                /* kJ/mol quartic wall constant (1e6) */
  const double *pH;             /* [R] */
  const uint64_t *replica_seed; /* [R] Philox keys */
  const double *lambda0;        /* [R*C] initial lambda or NULL (all 0 = protonated) */
  const float *pos_replicas;    /* [R*N*3] per-replica positions or NULL (system pos) */
  const float *vel_replicas;    /* [R*N*3] per-replica velocities or NULL (system vel) */
  int32_t frame_capacity;       /* lambda frames kept per replica between cph_get_frames (>=1) */
  void *cuda_stream;            /* cudaStream_t to launch on (NULL = legacy default) */
  void *(*dev_alloc)(size_t bytes, void *alloc_ctx);   /* NULL -> cudaMalloc */
  void (*dev_free)(void *ptr, void *alloc_ctx);
  void *alloc_ctx;
  /* Dynamic Barrier and Well Optimization.  Both off by default;
   * each can be enabled independently.  Block lengths must be
   * multiples of nstlist.  The rule constants default to the paper's values. */
  int32_t dbo_well;             /* 1: regulate the well centres */
  int32_t dbo_barrier;          /* 1: regulate the barrier heights */
  int64_t dbo_well_steps;       /* well block, steps (20000 = 40 ps) */
  int64_t dbo_barrier_steps;    /* barrier block, steps (500000 = 1 ns) */
  int64_t dbo_censor_steps;     /* censor window after an adjustment (5000 = 10 ps) */
  double dbo_well_near;         /* 0.2: lambda < 0.2 near well 0, lambda > 1 - 0.2 near well 1 */
  double dbo_residency;         /* 0.70: fraction of the block near one well to act */
  double dbo_well_tol;          /* 0.03: |mean - ideal| tolerance */
  double dbo_well_gain;         /* 0.5: shift = gain * (ideal - mean) */
  double dbo_well_cap;          /* 0.08: |accumulated shift| cap */
  double dbo_trans_lo;          /* 0.2 \  in transition: trans_lo < lambda < trans_hi */
  double dbo_trans_hi;          /* 0.8 /                                           */
  double dbo_target;            /* 0.25: target in-transition fraction */
  double dbo_target_tol;        /* 0.05 */
  double dbo_barrier_step;      /* 1.0 kJ/mol */
  double dbo_barrier_min;       /* 1 kJ/mol */
  double dbo_barrier_max;       /* 20 kJ/mol */
  /* Thermostat: 0 = Langevin BAOAB with gamma_atom / gamma_lambda (default);
   * 1 = Bussi-Donadio-Parrinello velocity rescaling as in the paper (PAPER.md:888,
   * :902-906), one group per replica for the atoms (3 x mobile atoms degrees of
   * freedom) and one for its lambda particles (C degrees of freedom), applied in the
   * middle of the step in place of the Langevin O step (R27, R28). */
  int32_t thermostat;
  double tau_atom;              /* ps (0.1) */
  double tau_lambda;            /* ps (1.0) */
  /* pH replica exchange (SURVEY §8(f) f3; the paper's outlook, PAPER.md:1664, :1738;
   * DESIGN.md R29, R30).  Replicas of all contexts taking part (one per GPU) form
   * remd_total / n_ph_levels ladders in global order (global replica g = remd_first + r
   * belongs to ladder g / n_ph_levels); every replica's pH must be one of ph_levels and
   * the labels inside a ladder a permutation of the levels.  Not combinable with DBO
   * or fixed-lambda mode (CPH_E_UNSUPPORTED). */
  int32_t n_ph_levels;          /* P >= 2 enables exchange; 0 = off */
  const double *ph_levels;      /* [P] strictly ascending pH levels */
  int32_t remd_first;           /* global index of this context's replica 0 (0) */
  int32_t remd_total;           /* replicas over all contexts, multiple of P (0 = R) */
  /* 0: charge interpolation (default, the north star's PME scheme); 1: Hamiltonian
   * interpolation, Eq. 1 literally (R31): E_coul of
   * the interpolated charges plus, per lambda-group, C = 1/4 sum_{s,t} w_s w_t D_st with
   * D_st = (q^s - q^t)^T G (q^s - q^t) over the group's atoms (real space, exclusion, self
   * and exact Ewald reciprocal terms); its lambda derivative is part of the Coulomb
   * dV/dlambda and its forces of the atom forces.  Groups of at most 32 atoms. */
  int32_t hamiltonian;
  /* 0: PME spread with fp32 atomics (default; runs agree to rounding); 1: the spread
   * accumulates in 64-bit fixed point (2^-40 e resolution, integer atomics commute), so the
   * whole Langevin step is bitwise reproducible run to run (SURVEY §5 optional fixed-point
   * accumulation); 64 integer atomics per atom instead of 16-32 float4 ones plus one grid
   * conversion pass. */
  int32_t deterministic;
  /* Replica sub-batches stepped concurrently (0 = automatic, the default; 1 = one batch).
   * The R replicas are split into S consecutive, near-equal batches, each with its own
   * device buffers, CUDA graph and stream; cph_step interleaves them in chunks of 32 nstlist
   * blocks, so one batch's PME chain (FFTs, solve, gather: few CTAs) runs under another's
   * pair kernel instead of leaving SMs idle at the end of every step.  Every random number
   * is keyed on (replica seed, step, atom) and every kernel works per replica, so results
   * are those of one batch up to rounding (identical trajectories in tests/test_gpu_subbatch.py).
   * Automatic: S = min(R, 4) when R * n_atoms >= 24000, else 1.  Every call
   * stays ordered on cph_get_stream(); per-replica getters route to the batch holding the
   * replica.  A call that fails part-way (e.g. a latched device error during cph_step) can
   * leave the batches at different steps: restore a checkpoint (cph_set_state_all) or
   * destroy the context. */
  int32_t sub_batches;
  /* Pair-list layout (ABI v5; 0 = automatic, the default).  1: a full per-atom Verlet list
   * (every pair in both atoms' rows; the pair kernel sums each atom's row in a fixed order
   * with no atomics).  2: a half cluster-pair list: super-clusters of 32 consecutive atoms of
   * a cell column against j-clusters of 4 consecutive sorted atoms, each entry carrying one
   * 32-bit interaction mask per 8-atom i-cluster whose bits are exactly the canonical pairs
   * (R14, exclusions removed, each unordered pair once); the pair kernel evaluates
   * a mask's pairs once and adds the j-side forces and potentials with float4 reductions.
   * Automatic = 1: on B200 the cluster kernel evaluates 757 pair slots per atom (8x4 masks
   * are 38 % full at r_list 1.1 nm) against 578 per-atom entries and is slower.
   * Both give the same pair set (cph_get_pairlist, bit-exact) and agree to rounding;
   * deterministic = 1 requires 0 or 1 (the j-side reductions of 2 are order-dependent,
   * CPH_E_INVALID). */
  int32_t pair_list;
} cph_params;

/* DBO event kinds (cph_dbo_event.kind) */
enum {
  CPH_DBO_WELL0 = 0,            /* centre of the lambda = 0 well moved */
  CPH_DBO_WELL1 = 1,            /* centre of the lambda = 1 well moved */
  CPH_DBO_BARRIER = 2,          /* barrier of a lambda_p coordinate */
  CPH_DBO_BARRIER_T_PROT = 3,   /* tautomer barrier used while protonated (lambda_p < 0.5) */
  CPH_DBO_BARRIER_T_DEPROT = 4  /* tautomer barrier used while deprotonated */
};

typedef struct {
  int64_t step;                 /* block-end step S; the new value applies from step S+1 */
  int32_t replica, coord, kind, pad;
  double old_value, new_value;  /* well centre (nm-free lambda units) or barrier kJ/mol */
} cph_dbo_event;

/* Fill *p with the defaults quoted above (pH/seed pointers NULL). */
void cph_default_params(cph_params *p);

/* Validate, copy to the device, run the PFC for every replica's pH, build the
 * pair list and evaluate forces/potentials/energies at step 0.  The pair-list
 * capacity per atom is 1.6x the mean neighbour count + 64, grown once here if the
 * initial configuration exceeds it; an overflow at a later rebuild is latched and
 * reported as CPH_E_STATE by the next call.
 * CPH_E_INVALID: non-finite input, bad sizes, a group whose total charge
 * varies with lambda, rlist >= min(box)/2, rc > rlist.
 * CPH_E_UNSUPPORTED: pme_order != 4, grid not even / not 2,3,5,7-smooth. */
cph_status cph_create(const cph_system *sys, const cph_params *params, cph_ctx **out);
void cph_destroy(cph_ctx *ctx);

/* Number of lambda coordinates C per replica and atoms N. */
int32_t cph_n_coords(const cph_ctx *ctx);
int32_t cph_n_atoms(const cph_ctx *ctx);
int32_t cph_n_replicas(const cph_ctx *ctx);
/* Number of replica sub-batches S the context steps concurrently (cph_params.sub_batches). */
int32_t cph_n_sub_batches(const cph_ctx *ctx);

/* The CUDA stream every call of this context enqueues on (the cph_params.cuda_stream the
 * caller passed, or the context's own non-blocking stream when that was NULL). */
void *cph_get_stream(const cph_ctx *ctx);
/* Change one replica's pH: recomputes the PFC well depths (host), uploads them and
 * re-evaluates dV_bias/dlambda and E_bias at the current lambda (the next half kick and
 * the getters see the new pH).  replica in [0, R). */
cph_status cph_set_pH(cph_ctx *ctx, int32_t replica, double pH);

/* Advance all replicas by n_steps >= 0 (asynchronous on the context stream). */
cph_status cph_step(cph_ctx *ctx, int64_t n_steps);

/* Block until the context stream is idle; reports latched device errors. */
cph_status cph_sync(cph_ctx *ctx);

/* Current step index (number of completed steps since create). */
int64_t cph_current_step(const cph_ctx *ctx);

/* Getters (synchronize first).  replica in [0, R). */
cph_status cph_get_lambdas(cph_ctx *ctx, int32_t replica, double *lam /*[C]*/, double *vel /*[C] or NULL*/);
/* dV/dlambda at the current state: Coulomb part f sum dq/dl phi, and bias part. */
cph_status cph_get_dvdl(cph_ctx *ctx, int32_t replica, double *coul /*[C]*/, double *bias /*[C]*/);
/* Energies at the current state in the CPH_E_* order; total = sum of the others. */
cph_status cph_get_energies(cph_ctx *ctx, int32_t replica, double *e /*[CPH_N_ETERMS]*/);
/* PFC results: lambda=1 well depth d1 per coordinate (kJ/mol). */
cph_status cph_get_bias_params(cph_ctx *ctx, int32_t replica, double *d1 /*[C]*/);
/* lambda frames recorded every nstout steps since the last call (oldest first);
 * buf [cap*C] floats; *n_frames = frames written; frames beyond capacity are
 * dropped oldest-first and *n_dropped reports how many. */
cph_status cph_get_frames(cph_ctx *ctx, int32_t replica, float *buf, int64_t cap,
                          int64_t *n_frames, int64_t *n_dropped);
/* As cph_get_frames, plus per frame the step it was taken at (steps [cap] or NULL),
 * the pH level index the replica simulated then (labels [cap] or NULL; -1 without
 * replica exchange)
 * and per frame and coordinate a censor flag (censored [cap*C] or NULL): 1 iff the
 * coordinate's site had a DBO adjustment at a block end S with
 * S < step <= S + dbo_censor_steps (R26). */
cph_status cph_get_frames_ex(cph_ctx *ctx, int32_t replica, float *buf, uint8_t *censored,
                             int64_t *steps, int32_t *labels, int64_t cap, int64_t *n_frames,
                             int64_t *n_dropped);
/* DBO parameters per coordinate [C*4]: (a0, a1, h_prot, h_deprot) = well centres of
 * the lambda = 0 and lambda = 1 wells, and the barrier heights (kJ/mol).  lambda_p
 * coordinates use h_prot == h_deprot; a tautomer coordinate's barrier is
 * h_prot + (h_deprot - h_prot) S(lambda_p), S the clamped smoothstep (R25).
 * Before any adjustment: (0, 1, barrier, barrier). */
cph_status cph_get_dbo_params(cph_ctx *ctx, int32_t replica, double *p);
/* Replace them (e.g. a restart): requires |a0| <= 0.2, |a1 - 1| <= 0.2, barriers in
 * (0, 100] and h_prot == h_deprot for lambda_p coordinates (else CPH_E_INVALID).
 * Re-runs the PFC of that replica and re-evaluates its forces; block accumulators
 * are kept. */
cph_status cph_set_dbo_params(cph_ctx *ctx, int32_t replica, const double *p);
/* Adjustment log since the last call (drained); *n = events written, up to cap;
 * the rest stay queued. */
cph_status cph_get_dbo_events(cph_ctx *ctx, cph_dbo_event *ev, int64_t cap, int64_t *n);
/* Current block accumulators of one replica: well [C*5] = (steps, steps near 0,
 * sum of lambda near 0, steps near 1, sum of lambda near 1); barrier [C*4] =
 * (frames A, in-transition A, frames B, in-transition B) with A = all frames for
 * lambda_p coordinates / protonated frames for tautomer coordinates, B =
 * deprotonated frames.  Either pointer may be NULL. */
cph_status cph_get_dbo_stats(cph_ctx *ctx, int32_t replica, double *well, double *barrier);

/* pH replica exchange (n_ph_levels >= 2).  One attempt = cph_exchange_energies on every
 * context, the rows of all contexts concatenated in global replica order (an NCCL
 * all-gather across GPUs), then cph_exchange_apply on every context with the same seed
 * and attempt index: each applies all Metropolis decisions (identical everywhere) to its
 * own replicas and re-evaluates their bias forces.  Call between cph_step calls.
 * rows / rows_all are DEVICE pointers on the context's device; the work is enqueued on
 * the context stream (no host synchronisation).
 * cph_exchange_energies: rows [R*(P+1)] = (label, E_0 .. E_{P-1}) per local replica,
 *   E_p = pH-dependent bias (VpH + Vdw at level p's PFC depths), kJ/mol, fp64.
 * cph_exchange_apply: rows_all [remd_total*(P+1)]; pairs (p, p+1), p = attempt mod 2,
 *   +2, ...; accept with min(1, exp(-Delta/kT)), u from Philox(seed; attempt, ladder, p, 5). */
/* Labels that do not form ladders (a level missing or held twice in a ladder, or out of
 * range) make cph_exchange_apply a no-op and latch CPH_E_STATE (reported by the next sync).
 * Ordering: both calls are enqueued on the context stream (cph_get_stream); a caller that
 * fills or reads the row buffers on another stream (e.g. NCCL on torch's current stream)
 * must order the two streams with events around the calls (the Python binding does). */
cph_status cph_exchange_energies(cph_ctx *ctx, double *rows);
cph_status cph_exchange_apply(cph_ctx *ctx, const double *rows_all, uint64_t seed, int64_t attempt);
/* Single-context shortcut (remd_total == R): energies + apply on an internal buffer. */
cph_status cph_exchange(cph_ctx *ctx, uint64_t seed, int64_t attempt);
/* Current level index per local replica [R] (synchronizes), and restart setter. */
cph_status cph_get_labels(cph_ctx *ctx, int32_t *labels);
cph_status cph_set_labels(cph_ctx *ctx, const int32_t *labels);
/* Attempts and accepted swaps per ladder and level pair [L*(P-1)], L = remd_total/P
 * (every context counts every ladder). */
cph_status cph_get_exchange_stats(cph_ctx *ctx, int64_t *attempts, int64_t *accepts);

/* Force on every atom [3N] (kJ mol^-1 nm^-1) and the full electrostatic potential
 * phi_i = (1/f) dE_coul/dq_i [N] (e/nm; real + exclusion + reciprocal + self +
 * net-charge terms), original order.  Either pointer may be NULL. */
cph_status cph_get_forces(cph_ctx *ctx, int32_t replica, float *f, float *phi);
/* Current positions [3N] and velocities [3N] (original order); either may be NULL. */
cph_status cph_get_positions(cph_ctx *ctx, int32_t replica, float *pos, float *vel);
/* Canonical pair list of the last rebuild: non-excluded pairs (i<j, original
 * indices) with float32 d^2 < rlist^2, lexicographically sorted, as [2*n].
 * If cap < n nothing is written and *n tells the size needed. */
cph_status cph_get_pairlist(cph_ctx *ctx, int32_t replica, int32_t *pairs, int64_t cap, int64_t *n);
/* Every directed entry (i, j) (original indices) the pair kernel evaluates from the last
 * rebuild's list, sorted lexicographically, as [2*n]; each canonical pair (i, j) of
 * cph_get_pairlist must appear exactly twice, as (i, j) and (j, i) (the kernel's list is
 * full, both directions; SURVEY §8(c) "pair lists bit-exact").  Same size protocol. */
cph_status cph_get_pairlist_directed(cph_ctx *ctx, int32_t replica, int32_t *pairs, int64_t cap, int64_t *n);
/* Rows of that directed list for selected atoms (for large systems): for atoms[k]
 * (original index) its partners j, sorted ascending, are cols[row_ptr[k] .. row_ptr[k+1]).
 * row_ptr [n_atoms+1] is always filled; cols [cap] only up to cap entries (call again with
 * cap >= row_ptr[n_atoms] to get all).  CPH_E_INVALID on an out-of-range atom. */
cph_status cph_get_pairlist_rows(cph_ctx *ctx, int32_t replica, const int32_t *atoms, int32_t n_atoms,
                                 int32_t *row_ptr, int32_t *cols, int64_t cap);
/* The device's lambda-group CSR mapped back to original atom indices (north star: lambda-group
 * indexing bit-exact): group_ptr / coord_ptr [G+1] as stored on the device; atoms[k] = the
 * original index reached from lambda slot k through the device's sorted-slot permutation
 * (iperm then meta); slot_atoms[k] = the original index of the sorted slot whose meta word
 * carries lambda slot k (-1 if none).  Both must equal the input group_atoms. */
cph_status cph_get_lambda_groups(cph_ctx *ctx, int32_t replica, int32_t *group_ptr, int32_t *coord_ptr,
                                 int32_t *atoms /*[n_lambda]*/, int32_t *slot_atoms /*[n_lambda]*/);
/* Fixed-lambda TI (mode 1): mean of the Coulomb dV/dlambda = f sum (dq/dl) phi per
 * coordinate over the steps completed since create or the last cph_set_state(_all)
 * (which restart the accumulators), and the number of samples; this is the
 * <dH_ref/dlambda> = <dV_coul/dlambda> the Vmm calibration fits. */
cph_status cph_get_ti_means(cph_ctx *ctx, int32_t replica, double *mean /*[C]*/, int64_t *n_samples);
/* Checkpoint of one replica: size query with buf == NULL (*n gets bytes).  The blob carries
 * the step (Philox counters, frame / nstlist / DBO phases count from it).  cph_set_state
 * (one replica) requires the blob's step to equal the context's current step
 * (CPH_E_STATE otherwise); cph_set_state_all (every replica) requires all blobs to carry
 * the same step and moves the context's clock to it, so a restore into a fresh context
 * continues the run. */
cph_status cph_get_state(cph_ctx *ctx, int32_t replica, void *buf, int64_t cap, int64_t *n);
cph_status cph_set_state(cph_ctx *ctx, int32_t replica, const void *buf, int64_t n);

/* All replicas at once (blob = R consecutive per-replica blobs of cph_get_state);
 * cph_set_state_all re-evaluates forces once for the whole batch.  A restore re-sorts the atoms
 * and rebuilds the pair list unless every restored atom is where the last rebuild put it
 * (minimum-image displacement <= 1e-5 nm): then that list is the list of the restored
 * configuration and is kept.  Headers and finiteness are checked before anything is
 * overwritten (CPH_E_INVALID, state unchanged); the re-evaluation is enqueued on the context
 * stream and not awaited, so a device-side failure in it is reported by the next call. */
cph_status cph_get_state_all(cph_ctx *ctx, void *buf, int64_t cap, int64_t *n);
cph_status cph_set_state_all(cph_ctx *ctx, const void *buf, int64_t n);

/* Run n_steps eagerly with CUDA events around every kernel class (serialised,
 * one stream) and return the summed milliseconds per class [CPH_N_KCLASSES]
 * and the number of launches per class [CPH_N_KCLASSES] (either may be NULL). */
cph_status cph_profile_steps(cph_ctx *ctx, int64_t n_steps, double *ms, int64_t *launches);
/* Number of kernel launches of this library issued so far (graph replays
 * counted per contained kernel; cuFFT's internal kernels not included). */
int64_t cph_launch_count(const cph_ctx *ctx);

const char *cph_last_error(const cph_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CPH_H */
