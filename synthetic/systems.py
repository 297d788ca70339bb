"""Deterministic synthetic constant-pH systems shaped like the paper's workloads.

Data only (see package docstring).  Recipe (DESIGN.md §"Input recipe"):

* Solvent: unbonded charged Lennard-Jones particles, number density
  rho = 100 nm^-3 (3-site-water pair density), mass 18 u, sigma 0.20 nm,
  eps 0.5 kJ/mol, charges +-0.2 e (equal counts, random assignment) on a
  jittered cubic lattice.
* Ions: 150 mM NaCl ("a salt concentration of 150~mM NaCl"),
  n_pairs = round(0.0903 * V[nm^3]); one extra Cl- per His-like site because
  positive initial states are neutralised by Cl- (PAPER.md:814-815).
* Solute: frozen (mass 0) residues; titratable Asp/Glu-like (7 atoms) and
  His-like (10 atoms) residues with state charges A..D,
  filler residues with random neutral charges; all intra-residue pairs are
  exclusions.
* Charge buffers: one frozen 3-site water per titratable site whose oxygen
  switches -0.834 -> +0.166 e, placed >= 2 nm from solute
  and other buffers where the box allows.
* Workload shapes (BASELINE.json configs): C1 capped Glu in 1.5k atoms,
  C2 GEAHG pentapeptide 7k, C3 cardiotoxin-V-like 25k, C4 lysozyme-like 40k,
  C5 membrane-channel-like 250k.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

KB = 0.0083144626  # kJ mol^-1 K^-1 (CODATA R / 1000), for Maxwell-Boltzmann draws only

# ---------------------------------------------------------------------------
# Residue templates: state charges (A, B, C, D) per atom, in e.
# Eq. 2: A/B protonated (lambda_p = 0), C/D deprotonated.
# 2-state sites use A = B and C = D.  His: A = B = HIP,
# C = HID (delta), D = HIE (epsilon).
# ---------------------------------------------------------------------------
_GLU_A = [0.10, -0.10, -0.05, 0.60, -0.55, -0.50, 0.50]     # sum 0
_GLU_C = [0.10, -0.10, -0.20, 0.60, -0.70, -0.70, 0.00]     # sum -1
_HIP = [0.13, 0.19, -0.51, 0.44, 0.32, 0.18, -0.51, 0.44, 0.19, 0.13]   # +1
_HID = [0.09, -0.05, -0.36, 0.32, 0.25, 0.13, -0.70, 0.00, 0.22, 0.10]   # 0
_HIE = [0.10, 0.22, -0.70, 0.00, 0.25, 0.13, -0.36, 0.32, -0.05, 0.09]   # 0

# reference pKa (Table 2): macro, micro-delta, micro-eps
PKA_ASP = (4.00, 4.00, 4.00)
PKA_GLU = (4.40, 4.40, 4.40)
PKA_HIS = (6.38, 6.53, 6.92)

# LJ types: 0 solvent/buffer, 1 Na+, 2 Cl-, 3 solute heavy atom
_SIGMA = np.array([0.20, 0.25, 0.40, 0.25])
_EPS = np.array([0.50, 0.50, 0.50, 0.30])
T_SOLVENT, T_NA, T_CL, T_SOLUTE = 0, 1, 2, 3

BUFFER_O_Q = (-0.834, 0.166)
BUFFER_H_Q = 0.417

DEFAULT_PARAMS = dict(
    rc=1.0, rlist=1.1, ewald_rtol=1e-5, pme_order=4, nstlist=10,
    nstout=250, nstenergy=250, dt=0.002, temperature=300.0,
    gamma_atom=1.0, gamma_lambda=1.0, lambda_mass=60.0,
    barrier=6.0, wall_k=1e6,
)


@dataclass
class SyntheticSystem:
    name: str
    box: np.ndarray            # (3,) f64, nm
    pos: np.ndarray            # (N,3) f32, nm
    mass: np.ndarray           # (N,) f32, u; 0 = frozen
    charge: np.ndarray         # (N,) f32, e (lambda atoms: state-A value, not used)
    type: np.ndarray           # (N,) i32
    c6: np.ndarray             # (T,T) f64 kJ mol^-1 nm^6
    c12: np.ndarray            # (T,T) f64 kJ mol^-1 nm^12
    excl: np.ndarray           # (n_excl,2) i32, i<j
    group_kind: np.ndarray     # (G,) i32: 2 or 3 states
    group_ptr: np.ndarray      # (G+1,) i32
    group_atoms: np.ndarray    # (n_lambda,) i32
    state_q: np.ndarray        # (n_lambda,4) f64
    is_buffer: np.ndarray      # (n_lambda,) i32
    pKa: np.ndarray            # (G,3) f64 macro, delta, eps
    vmm: np.ndarray            # (G,36) f64, c[a*6+b] for lambda_p^a lambda_t^b
    pme_grid: tuple
    params: dict = field(default_factory=lambda: dict(DEFAULT_PARAMS))
    pH_grid: tuple = ()

    @property
    def n_atoms(self):
        return int(self.pos.shape[0])

    @property
    def n_groups(self):
        return int(self.group_kind.shape[0])

    @property
    def n_coords(self):
        return int(sum(1 if k == 2 else 2 for k in self.group_kind))


CONFIGS = {
    # cfg: (name, N target, box L, K, residues spec, pH grid)
    1: dict(name="C1_glu_1.5k", n=1500, L=2.466, K=24, shape="single",
            sites=["E"], fillers=0, pH=(4.40,)),
    2: dict(name="C2_GEAHG_7k", n=7000, L=4.121, K=40, shape="chain",
            sites=["E", "H"], fillers=3, order=("F", "E", "F", "H", "F"),
            pH=(2.0, 2.5, 3.0, 3.25, 3.5, 3.75, 4.0, 4.5, 5.0, 5.5, 6.0, 6.25,
                6.5, 6.75, 7.0, 7.5, 8.0)),
    3: dict(name="C3_cardiotoxinV_25k", n=25000, L=6.300, K=60, shape="blob",
            sites=["D"] * 5 + ["E"] * 5 + ["H"] * 5, fillers=45,
            pH=tuple(np.arange(1.0, 8.01, 0.5).round(2))),
    4: dict(name="C4_lysozyme_40k", n=40000, L=7.368, K=72, shape="blob",
            sites=["D"] * 8 + ["E"] * 8 + ["H"] * 4, fillers=109,
            pH=tuple(np.arange(-1.0, 9.01, 0.5).round(2))),
    5: dict(name="C5_channel_250k", n=250000, L=13.572, K=128, shape="channel",
            sites=["D"] * 60 + ["E"] * 60 + ["H"] * 30, fillers=450,
            pH=(2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0, 9.0)),
}


def replica_seeds(cfg: int, n: int, base: int = 0) -> np.ndarray:
    """64-bit replica seeds = hash(cfg, replica index, base)."""
    out = []
    for r in range(n):
        h = hashlib.sha256(f"cph-{cfg}-{base}-{r}".encode()).digest()
        out.append(int.from_bytes(h[:8], "little"))
    return np.array(out, dtype=np.uint64)


def _lj_tables():
    T = len(_SIGMA)
    c6 = np.zeros((T, T))
    c12 = np.zeros((T, T))
    for a in range(T):
        for b in range(T):
            s = 0.5 * (_SIGMA[a] + _SIGMA[b])      # Lorentz-Berthelot mixing
            e = np.sqrt(_EPS[a] * _EPS[b])
            c6[a, b] = 4.0 * e * s ** 6
            c12[a, b] = 4.0 * e * s ** 12
    return c6, c12


def _residue_geometry(rng, n_atoms, center, radius=0.22, dmin=0.11):
    pts = []
    tries = 0
    while len(pts) < n_atoms:
        tries += 1
        p = center + rng.uniform(-radius, radius, 3)
        if np.linalg.norm(p - center) > radius:
            continue
        if all(np.linalg.norm(p - q) >= dmin for q in pts) or tries > 5000:
            pts.append(p)
    return np.array(pts)


def _residue_centers(rng, cfg, n_res, L):
    c = np.full(3, L / 2.0)
    shape = cfg["shape"]
    if shape == "single":
        return [c.copy()]
    centers = []
    if shape == "chain":
        # extended chain along x through the box center (PAPER.md:1111-1113 straight chain)
        for k in range(n_res):
            centers.append(c + np.array([(k - (n_res - 1) / 2) * 0.38, 0.0, 0.0]))
        return centers
    dmin = 0.52
    if shape == "blob":
        R = 0.62 * (n_res ** (1.0 / 3.0)) * 0.55 + 0.4
        gen = lambda: c + rng.uniform(-R, R, 3)
        ok = lambda p: np.linalg.norm(p - c) <= R
    else:  # channel: cylindrical shell of residues along z
        Rin, Rout, H = 1.2, 2.6, 0.8 * L
        def gen():
            r = rng.uniform(Rin, Rout)
            t = rng.uniform(0, 2 * np.pi)
            z = rng.uniform(-H / 2, H / 2)
            return c + np.array([r * np.cos(t), r * np.sin(t), z])
        ok = lambda p: True
    tries = 0
    while len(centers) < n_res:
        tries += 1
        p = gen()
        if not ok(p):
            continue
        if tries < 200000 and centers and np.min(np.linalg.norm(np.array(centers) - p, axis=1)) < dmin:
            continue
        centers.append(p)
    return centers


def _min_image_dist(a, b, L):
    d = a[None, :] - b
    d -= L * np.round(d / L)
    return np.sqrt((d * d).sum(-1))


def make_system(cfg: int, seed: int | None = None, n_target: int | None = None) -> SyntheticSystem:
    """Build configuration `cfg` (1..5) deterministically from `seed` (default 1000*cfg)."""
    spec = CONFIGS[cfg]
    rng = np.random.default_rng(1000 * cfg if seed is None else seed)
    # the box edge is an fp32 value: the device stores and wraps coordinates in fp32 with
    # fl32(L), so the oracle (fp64) and the device then simulate the same box (R34)
    L = float(np.float32(spec["L"]))
    n_target = spec["n"] if n_target is None else n_target
    box = np.array([L, L, L], dtype=np.float64)

    pos, mass, charge, typ = [], [], [], []
    excl = []
    g_kind, g_ptr, g_atoms, g_q, g_buf, g_pka = [], [0], [], [], [], []

    site_list = list(spec["sites"])
    n_res = len(site_list) + spec["fillers"]
    # interleave sites among residues (pentapeptide order G E A H G for C2)
    if "order" in spec:
        order = list(spec["order"])
    elif spec["shape"] == "chain":
        order = site_list + ["F"] * spec["fillers"]
    else:
        order = site_list + ["F"] * spec["fillers"]
        rng.shuffle(order)
    centers = _residue_centers(rng, spec, n_res, L)

    def add_atom(p, m, q, t):
        pos.append(np.asarray(p, dtype=np.float64))
        mass.append(m)
        charge.append(q)
        typ.append(t)
        return len(pos) - 1

    site_atoms_centers = []
    for kind, cen in zip(order, centers):
        if kind == "F":
            na = 8
            q = rng.uniform(-0.4, 0.4, na)
            q -= q.mean()
            xyz = _residue_geometry(rng, na, cen)
            idx = [add_atom(xyz[a], 0.0, q[a], T_SOLUTE) for a in range(na)]
        else:
            if kind in ("D", "E"):
                qa, qc = _GLU_A, _GLU_C
                states = [(qa[a], qa[a], qc[a], qc[a]) for a in range(len(qa))]
                pk = PKA_ASP if kind == "D" else PKA_GLU
                g_kind.append(2)
            else:
                states = [(_HIP[a], _HIP[a], _HID[a], _HIE[a]) for a in range(len(_HIP))]
                pk = PKA_HIS
                g_kind.append(3)
            na = len(states)
            xyz = _residue_geometry(rng, na, cen)
            idx = [add_atom(xyz[a], 0.0, states[a][0], T_SOLUTE) for a in range(na)]
            g_atoms.extend(idx)
            g_q.extend(states)
            g_buf.extend([0] * na)
            g_pka.append(pk)
            site_atoms_centers.append(len(g_kind) - 1)
            g_ptr.append(None)  # fixed up when buffer added
        for a in range(len(idx)):
            for b in range(a + 1, len(idx)):
                excl.append((idx[a], idx[b]))

    solute_xyz = np.array(pos)
    # --- charge buffers: one per titratable site -------------------------------------
    buffers = []
    n_sites = len(g_kind)
    buf_atoms_per_site = []
    for s in range(n_sites):
        best, best_d = None, -1.0
        for _ in range(3000):
            p = rng.uniform(0, L, 3)
            d = np.min(_min_image_dist(p, solute_xyz, L))
            if buffers:
                d = min(d, np.min(_min_image_dist(p, np.array(buffers), L)))
            if d > best_d:
                best, best_d = p, d
            if d >= 2.0:
                break
        buffers.append(best)
        o = add_atom(best, 0.0, BUFFER_O_Q[0], T_SOLVENT)
        h1 = add_atom(best + np.array([0.0957, 0.0, 0.0]), 0.0, BUFFER_H_Q, T_SOLVENT)
        h2 = add_atom(best + np.array([-0.024, 0.0927, 0.0]), 0.0, BUFFER_H_Q, T_SOLVENT)
        excl.extend([(o, h1), (o, h2), (h1, h2)])
        buf_atoms_per_site.append(o)

    # assemble lambda-group CSR: site atoms followed by the buffer oxygen
    site_atom_lists = []
    cursor = 0
    for s in range(n_sites):
        na = 7 if g_kind[s] == 2 else 10
        site_atom_lists.append((cursor, cursor + na))
        cursor += na
    atoms_csr, q_csr, buf_csr = [], [], []
    ptr = [0]
    for s in range(n_sites):
        a0, a1 = site_atom_lists[s]
        atoms_csr.extend(g_atoms[a0:a1])
        q_csr.extend(g_q[a0:a1])
        buf_csr.extend([0] * (a1 - a0))
        atoms_csr.append(buf_atoms_per_site[s])
        q_csr.append((BUFFER_O_Q[0], BUFFER_O_Q[0], BUFFER_O_Q[1], BUFFER_O_Q[1]))
        buf_csr.append(1)
        ptr.append(len(atoms_csr))

    fixed_xyz = np.array(pos)
    # --- mobile particles: solvent + ions on a jittered lattice ----------------------
    n_his = sum(1 for k in g_kind if k == 3)
    n_nacl = int(round(0.0903 * L ** 3))
    n_fixed = len(pos)
    n_mobile = n_target - n_fixed
    n_solv = n_mobile - 2 * n_nacl - n_his
    if n_solv % 2:
        n_solv -= 1
    n_mobile = n_solv + 2 * n_nacl + n_his
    # smallest cubic lattice that still has n_mobile free sites: spacing ~ rho^-1/3, so the
    # initial configuration has no LJ overlaps (sigma 0.2 nm vs spacing >= 0.21 nm)
    nside = int(np.ceil(n_mobile ** (1.0 / 3.0)))
    while True:
        a = L / nside
        g = (np.arange(nside) + 0.5) * a
        lat = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
        keep = np.ones((nside, nside, nside), bool)
        rad = int(np.ceil(0.24 / a)) + 1
        offs = np.arange(-rad, rad + 1)
        for p in fixed_xyz:
            c = np.floor(np.mod(p, L) / a).astype(int)
            ix = [(c[d] + offs) % nside for d in range(3)]
            sub = np.stack(np.meshgrid(*ix, indexing="ij"), -1).reshape(-1, 3)
            d = (sub + 0.5) * a - p
            d -= L * np.round(d / L)
            close = (d * d).sum(-1) < 0.24 ** 2
            keep[sub[close, 0], sub[close, 1], sub[close, 2]] = False
        lat = lat[keep.reshape(-1)]
        if len(lat) >= n_mobile:
            break
        nside += 1
    sel = rng.choice(len(lat), size=n_mobile, replace=False)
    sites = lat[sel] + rng.uniform(-0.01, 0.01, (n_mobile, 3))
    kinds = ([("Na", 22.99, 1.0, T_NA)] * n_nacl + [("Cl", 35.45, -1.0, T_CL)] * (n_nacl + n_his))
    solv_q = np.array([0.2] * (n_solv // 2) + [-0.2] * (n_solv // 2))
    rng.shuffle(solv_q)
    kinds += [("W", 18.0, float(q), T_SOLVENT) for q in solv_q]
    order_m = rng.permutation(n_mobile)
    for k, si in zip(kinds, order_m):
        add_atom(sites[si], k[1], k[2], k[3])

    P = np.array(pos)
    P = np.mod(P, L)
    c6, c12 = _lj_tables()
    excl_arr = np.array(sorted((min(i, j), max(i, j)) for i, j in excl), dtype=np.int32).reshape(-1, 2)
    G = n_sites
    vmm = rng.normal(0.0, 1.0, (G, 36))
    return SyntheticSystem(
        name=spec["name"], box=box, pos=P.astype(np.float32),
        mass=np.array(mass, np.float32), charge=np.array(charge, np.float32),
        type=np.array(typ, np.int32), c6=c6, c12=c12, excl=excl_arr,
        group_kind=np.array(g_kind, np.int32), group_ptr=np.array(ptr, np.int32),
        group_atoms=np.array(atoms_csr, np.int32), state_q=np.array(q_csr, np.float64),
        is_buffer=np.array(buf_csr, np.int32), pKa=np.array(g_pka, np.float64).reshape(-1, 3),
        vmm=vmm, pme_grid=(spec["K"],) * 3, params=dict(DEFAULT_PARAMS), pH_grid=tuple(spec["pH"]),
    )


def make_velocities(sys: SyntheticSystem, seed: int, temperature: float = 300.0) -> np.ndarray:
    """Maxwell-Boltzmann velocities (nm/ps), zero for frozen atoms; data only."""
    rng = np.random.default_rng(seed)
    m = sys.mass.astype(np.float64)
    sd = np.sqrt(np.where(m > 0, KB * temperature / np.where(m > 0, m, 1.0), 0.0))
    return (rng.normal(size=(sys.n_atoms, 3)) * sd[:, None]).astype(np.float32)


def random_lambdas(sys: SyntheticSystem, seed: int, lo: float = -0.1, hi: float = 1.1) -> np.ndarray:
    """Random lambda coordinates (for snapshot parity tests)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, sys.n_coords)


def small_system(n_solvent: int = 200, L: float = 2.3, seed: int = 7, his: bool = True) -> SyntheticSystem:
    """A few-hundred-atom system with one Glu-like and (optionally) one His-like site,
    for oracle self-tests and fast GPU parity cases (spans several tiles + ragged tail)."""
    rng = np.random.default_rng(seed)
    sysd = dict(name="tiny", n=0, L=L, K=20, shape="chain", sites=["E", "H"] if his else ["E"],
                fillers=0, pH=(4.4,))
    CONFIGS[-1] = sysd
    try:
        order_n = 7 + (10 if his else 0) + 3 * (2 if his else 1) + (1 if his else 0)
        s = make_system(-1, seed=seed, n_target=order_n + n_solvent)
    finally:
        del CONFIGS[-1]
    s.pme_grid = (20, 20, 20)
    s.name = "tiny"
    return s
