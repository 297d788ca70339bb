"""One constant-pH replica: energy/potential/dV/dlambda evaluation and the BAOAB step.

Follows, in order:
  * charges q(lambda) by Eq. 2 (oracle.charges)
  * E_coul = E_real + E_excl + E_self + E_net + E_rec, phi_i = (1/f) dE_coul/dq_i
    (oracle.ewald, oracle.pme)
  * dV/dlambda_k = f sum_{i in grp k} (dq_i/dlambda_k) phi_i + dV_bias/dlambda_k
    (F_lambda = -dH/dlambda; Eq. 3 bias, oracle.bias)
  * BAOAB (reading R9; velocity Verlet PAPER.md:896 + stochastic thermostat
    PAPER.md:902-907): B v+=dt/2 F/m; A x+=dt/2 v; O v=c1 v+sqrt((1-c1^2)kT/m) xi;
    A x+=dt/2 v; forces at (x, lambda) jointly; B v+=dt/2 F/m; c1 = exp(-gamma dt).
    With params thermostat="bussi" the O step is the Bussi velocity rescaling of the
    group (atoms tau_atom = 0.1 ps, lambda tau_lambda = 1 ps; PAPER.md:888, :902-906;
    oracle.thermostat, readings R27/R28).
  * Optional Hamiltonian interpolation (params hamiltonian=True; oracle.hamiltonian,
    PAPER.md:597-600): E_coul + sum_g C_g, its lambda derivative added to dvdl_coul and its
    forces to F (energy term "hi").
    Atoms: m from the system, mass 0 = frozen.  lambda: m = 60 u,
    gamma = 1/tau = 1 ps^-1.  Noise from oracle.philox.
  * Partition Function Correction at construction.
  * Optional DBO (oracle.dbo): statistics after every completed step;
    at the end of a block step S the rules run, the PFC is recomputed for the adjusted
    sites and the forces are re-evaluated at the unchanged (x, lambda),
    so step S+1 starts on the new bias.
"""
import math

import numpy as np

from . import bias as B
from . import dbo as DBO
from . import pfc as PFC
from . import thermostat as TH
from . import hamiltonian as HI
from .charges import charges, coord_ptr
from .ewald import (ewald_beta, exclusion_correction, net_charge_term, real_space,
                    recip_direct, self_term)
from .philox import normals
from .pme import pme
from .units import F_COUL, kT

ENERGY_TERMS = ("LJ", "real", "excl", "self", "recip", "net", "hi", "bias", "KE_atoms", "KE_lambda", "total")


class OracleReplica:
    def __init__(self, sys, pH, seed, lam0=None, vel0=None, pos0=None, params=None,
                 recip="pme", nmax=None, fixed_lambda=False, dbo=None, dbo_params=None):
        self.sys = sys
        p = dict(sys.params)
        if params:
            p.update(params)
        self.p = p
        self.pH = float(pH)
        self.seed = int(seed)
        self.box = np.asarray(sys.box, np.float64)
        self.beta = ewald_beta(p["rc"], p["ewald_rtol"])
        self.recip = recip
        self.nmax = nmax
        self.K = tuple(sys.pme_grid)
        self.fixed_lambda = fixed_lambda
        self.mass = sys.mass.astype(np.float64)
        self.mobile = self.mass > 0
        self.x = np.asarray(sys.pos if pos0 is None else pos0, np.float64).copy()
        self.v = np.zeros_like(self.x) if vel0 is None else np.asarray(vel0, np.float64).copy()
        self.v[~self.mobile] = 0.0
        self.cptr = coord_ptr(sys.group_kind)
        C = int(self.cptr[-1])
        self.lam = np.zeros(C) if lam0 is None else np.asarray(lam0, np.float64).copy()
        self.lamv = np.zeros(C)
        self.step_index = 0
        # DBO: per-coordinate (a0, a1, h_prot, h_deprot); config keys well, barrier (bool),
        # well_steps, barrier_steps, censor_steps
        self.dbo = dict(well=False, barrier=False, well_steps=20000, barrier_steps=500000, censor_steps=5000)
        if dbo:
            self.dbo.update(dbo)
        self.dbo_params = B.default_dbo(p["barrier"], C) if dbo_params is None else np.array(dbo_params, np.float64)
        self.lp_of = np.full(C, -1)
        for g, kind in enumerate(sys.group_kind):
            if int(kind) == 3:
                self.lp_of[self.cptr[g] + 1] = self.cptr[g]
        self.stats_well = DBO.BlockStats(C)
        self.stats_barrier = DBO.BlockStats(C)
        self.events = []              # (step, coord, kind, old, new)
        self.censor = []              # (group, step S): frames S < t <= S + censor_steps
        self.set_pH(pH)
        self.cur = self.evaluate(self.x, self.lam)

    # -- bias parameters (PFC) ---------------------------------------------------------
    def set_pH(self, pH):
        p = self.p
        self.pH = float(pH)
        self.d1 = np.zeros(int(self.cptr[-1]))
        for g in range(len(self.sys.group_kind)):
            self._pfc_group(g)

    def _pfc_group(self, g):
        p = self.p
        c0 = self.cptr[g]
        db = self.dbo_params
        if int(self.sys.group_kind[g]) == 2:
            self.d1[c0] = PFC.pfc_2state(db[c0, 2], self.sys.pKa[g, 0], self.pH, p["temperature"], p["wall_k"],
                                         db[c0, 0], db[c0, 1])
        else:
            self.d1[c0], self.d1[c0 + 1] = PFC.pfc_3state(db[c0, 2], self.sys.pKa[g], self.pH, p["temperature"],
                                                          p["wall_k"], db[c0:c0 + 2])

    def set_dbo_params(self, dbo_params):
        """Replace the DBO parameters, recompute the PFC and the forces."""
        self.dbo_params = np.array(dbo_params, np.float64)
        self.set_pH(self.pH)
        self.cur = self.evaluate(self.x, self.lam)

    def _dbo_block_end(self):
        S = self.step_index
        ev = []
        if self.dbo["well"] and S % self.dbo["well_steps"] == 0:
            ev += DBO.well_update(self.dbo_params, self.stats_well)
            self.stats_well = DBO.BlockStats(len(self.lam))
        if self.dbo["barrier"] and S % self.dbo["barrier_steps"] == 0:
            ev += DBO.barrier_update(self.dbo_params, self.stats_barrier, self.lp_of)
            self.stats_barrier = DBO.BlockStats(len(self.lam))
        if not ev:
            return
        groups = sorted({int(np.searchsorted(self.cptr, c, side="right") - 1) for c, *_ in ev})
        for c, kind, old, new in ev:
            self.events.append((S, c, kind, old, new))
        for g in groups:
            self._pfc_group(g)
            self.censor.append((g, S))
        self.cur = self.evaluate(self.x, self.lam)

    def bias(self, lam):
        p = self.p
        E = 0.0
        dv = np.zeros(len(lam))
        for g, kind in enumerate(self.sys.group_kind):
            c0 = self.cptr[g]
            lp = lam[c0]
            lt = lam[c0 + 1] if int(kind) == 3 else 0.0
            d1t = self.d1[c0 + 1] if int(kind) == 3 else 0.0
            nc = 2 if int(kind) == 3 else 1
            v, dp, dt = B.group_bias(kind, self.sys.vmm[g], self.sys.pKa[g], self.pH, p["temperature"],
                                     p["barrier"], self.d1[c0], d1t, p["wall_k"], lp, lt,
                                     self.dbo_params[c0:c0 + nc])
            E += v
            dv[c0] += dp
            if int(kind) == 3:
                dv[c0 + 1] += dt
        return E, dv

    # -- force / potential evaluation --------------------------------------------------
    def evaluate(self, x, lam):
        s, p = self.sys, self.p
        q, dq = charges(s, lam)
        rs = real_space(x, q, s.type, s.c6, s.c12, self.box, p["rc"], self.beta, s.excl,
                        max_chunks=p.get("sample_real_chunks"))    # bench.py CPU sample only
        ex = exclusion_correction(x, q, self.box, self.beta, s.excl)
        e_self, phi_self = self_term(q, self.beta)
        e_net, phi_net = net_charge_term(q, self.box, self.beta)
        if self.recip == "pme":
            rec = pme(x, q, self.box, self.beta, self.K, p["pme_order"])
            e_rec, phi_rec, f_rec = rec["E_rec"], rec["phi"], rec["F"]
        else:
            e_rec, phi_rec, f_rec = recip_direct(x, q, self.box, self.beta, self.nmax)
        phi = rs["phi"] + ex["phi"] + phi_rec + phi_self + phi_net
        F = rs["F"] + ex["F"] + f_rec
        C = len(lam)
        dvdl_coul = np.zeros(C)
        term_mag = np.zeros(C)
        for g, kind in enumerate(s.group_kind):
            c0 = self.cptr[g]
            for k in range(s.group_ptr[g], s.group_ptr[g + 1]):
                i = s.group_atoms[k]
                dvdl_coul[c0] += F_COUL * dq[k, 0] * phi[i]
                term_mag[c0] += abs(F_COUL * dq[k, 0] * phi[i])
                if int(kind) == 3:
                    dvdl_coul[c0 + 1] += F_COUL * dq[k, 1] * phi[i]
                    term_mag[c0 + 1] += abs(F_COUL * dq[k, 1] * phi[i])
        e_bias, dvdl_bias = self.bias(lam)
        e_hi = 0.0
        if p.get("hamiltonian", False):
            if getattr(self, "_kv", None) is None:
                self._kv = HI.kvectors(self.box, self.beta)
            e_hi, dv_hi, f_hi = HI.hi_terms(s, x, lam, self.cptr, self.box, self.beta, p["rc"], self._kv)
            dvdl_coul = dvdl_coul + dv_hi
            term_mag = term_mag + np.abs(dv_hi)
            F = F + f_hi
        return dict(q=q, phi=phi, F=F, dvdl_coul=dvdl_coul, dvdl_bias=dvdl_bias, term_mag=term_mag,
                    E=dict(LJ=rs["E_LJ"], real=rs["E_real"], excl=ex["E_excl"], self=e_self,
                           recip=e_rec, net=e_net, hi=e_hi, bias=e_bias),
                    phi_parts=dict(real=rs["phi"], excl=ex["phi"], recip=phi_rec, self=phi_self, net=phi_net))

    def energies(self):
        E = dict(self.cur["E"])
        E["KE_atoms"] = 0.5 * float(np.sum(self.mass[:, None] * self.v * self.v))
        E["KE_lambda"] = 0.5 * self.p["lambda_mass"] * float(np.sum(self.lamv ** 2))
        E["total"] = sum(E[k] for k in ENERGY_TERMS[:-1])
        return E

    # -- BAOAB -------------------------------------------------------------------------
    def step(self):
        p = self.p
        h = p["dt"]
        kt = kT(p["temperature"])
        n = self.step_index
        m = np.where(self.mobile, self.mass, 1.0)[:, None]
        mob = self.mobile[:, None]
        bussi = p.get("thermostat", "langevin") == "bussi"
        F = self.cur["F"]
        v = self.v + np.where(mob, 0.5 * h * F / m, 0.0)                  # B
        x = self.x + np.where(mob, 0.5 * h * v, 0.0)                      # A
        if bussi:                                                         # O: Bussi rescale
            nf = 3 * int(np.count_nonzero(self.mobile))
            K = 0.5 * float(np.sum(np.where(mob, m * v * v, 0.0)))
            R1, S = TH.bussi_draws(self.seed, n, TH.STREAM_ATOMS, nf)
            v = TH.bussi_alpha(K, nf, kt, h, p.get("tau_atom", 0.1), R1, S) * v
        else:                                                             # O: Langevin
            c1 = math.exp(-p["gamma_atom"] * h)
            sd = np.sqrt((1.0 - c1 * c1) * kt / m)
            xi = normals(self.seed, n, np.arange(len(self.x)), 0)[:, :3]
            v = np.where(mob, c1 * v + sd * xi, 0.0)
        x = x + np.where(mob, 0.5 * h * v, 0.0)                           # A
        lam, lamv = self.lam, self.lamv
        if not self.fixed_lambda:
            ml = p["lambda_mass"]
            Fl = -(self.cur["dvdl_coul"] + self.cur["dvdl_bias"])
            lamv = lamv + 0.5 * h * Fl / ml
            lam = lam + 0.5 * h * lamv
            if bussi:
                nf = len(lam)
                R1, S = TH.bussi_draws(self.seed, n, TH.STREAM_LAMBDA, nf)
                lamv = TH.bussi_alpha(0.5 * ml * float(np.sum(lamv * lamv)), nf, kt, h,
                                      p.get("tau_lambda", 1.0), R1, S) * lamv
            else:
                cl = math.exp(-p["gamma_lambda"] * h)
                sdl = math.sqrt((1.0 - cl * cl) * kt / ml)
                xil = normals(self.seed, n, np.arange(len(lam)), 1)[:, 0]
                lamv = cl * lamv + sdl * xil
            lam = lam + 0.5 * h * lamv
        cur = self.evaluate(x, lam)                                       # forces at (x, lambda)
        v = v + np.where(mob, 0.5 * h * cur["F"] / m, 0.0)                # B
        if not self.fixed_lambda:
            lamv = lamv + 0.5 * h * (-(cur["dvdl_coul"] + cur["dvdl_bias"])) / p["lambda_mass"]
        self.x, self.v, self.lam, self.lamv, self.cur = x, v, lam, lamv, cur
        self.step_index = n + 1
        if not self.fixed_lambda and (self.dbo["well"] or self.dbo["barrier"]):
            self.stats_well.add(self.lam, self.lp_of)
            self.stats_barrier.add(self.lam, self.lp_of)
            self._dbo_block_end()
