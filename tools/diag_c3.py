"""Diagnostic: per-coordinate dV/dlambda error budget at C3 (which lambda atoms / terms)."""
import numpy as np
import paper_2410_01626_b200 as cph
from oracle import ewald as OE
from oracle import pme as OP
from oracle.charges import charges, coord_ptr
from oracle.units import F_COUL
from synthetic.systems import make_system

s = make_system(3)
lam0 = np.random.default_rng(2).uniform(0, 1, (1, s.n_coords))
ctx = cph.cph_create(s, [5.0], [11], lambda0=lam0)
f, phi = ctx.cph_get_forces(0)
coul, _ = ctx.cph_get_dvdl(0)
q, dq = charges(s, lam0[0])
beta = OE.ewald_beta(1.0, 1e-5)
x = s.pos.astype(np.float64)
rec = OP.pme(x, q, s.box, beta, s.pme_grid, 4)
idx = np.unique(s.group_atoms)
phr, Fr = OE.real_space_at(idx, x, q, s.type, s.c6, s.c12, s.box, 1.0, beta, s.excl)
ex = OE.exclusion_correction(x, q, s.box, beta, s.excl)
_, phis = OE.self_term(q, beta)
_, phin = OE.net_charge_term(q, s.box, beta)
pos = {a: k for k, a in enumerate(idx)}
phi_ref = phr + ex["phi"][idx] + rec["phi"][idx] + phis[idx] + phin[idx]
d = phi[idx] - phi_ref
print("lambda-atom phi: max |err|", np.abs(d).max(), "rms phi", np.sqrt(np.mean(phi_ref ** 2)),
      "max rel", (np.abs(d) / np.abs(phi_ref)).max())
k = np.argmax(np.abs(d))
print("worst atom", idx[k], "phi_ref", phi_ref[k], "parts real", phr[k], "excl", ex["phi"][idx][k], "rec",
      rec["phi"][idx][k], "self", phis[idx][k], "net", phin[idx][k], "gpu", phi[idx][k])
cp = coord_ptr(s.group_kind)
for g in range(s.n_groups):
    ref = mag = 0.0
    for kk in range(s.group_ptr[g], s.group_ptr[g + 1]):
        p = phi_ref[pos[s.group_atoms[kk]]]
        ref += F_COUL * dq[kk, 0] * p
        mag += abs(F_COUL * dq[kk, 0] * p)
    e = abs(coul[cp[g]] - ref) / max(abs(ref), mag)
    if e > 5e-6:
        print("group", g, "kind", s.group_kind[g], "dvdl gpu", coul[cp[g]], "ref", ref, "mag", mag, "rel", e)
