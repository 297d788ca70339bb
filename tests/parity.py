"""Parity metrics of SURVEY §8(c) / DESIGN.md (shared by the GPU tests and bench checks)."""
import numpy as np

RTOL = 2e-5        # potentials, forces, dV/dlambda (north star)
ETOL = 1e-6        # total energy (north star)
POT_TERMS = ("LJ", "real", "excl", "self", "recip", "net", "hi", "bias")


def force_err(f_gpu, f_ref):
    return float(np.linalg.norm(np.asarray(f_gpu, np.float64) - f_ref) / np.linalg.norm(f_ref))


def phi_err(p_gpu, p_ref):
    return float(np.linalg.norm(np.asarray(p_gpu, np.float64) - p_ref) / np.linalg.norm(p_ref))


def force_atom_err(f_gpu, f_ref):
    """max_i |dF_i| / max(|F_i|, rms_i |F_i|): a single wrong atom (e.g. a dropped exclusion)
    cannot hide behind the norm-wise ratio."""
    f_ref = np.asarray(f_ref, np.float64)
    d = np.linalg.norm(np.asarray(f_gpu, np.float64) - f_ref, axis=1)
    mag = np.linalg.norm(f_ref, axis=1)
    rms = np.sqrt(np.mean(mag ** 2))
    return float(np.max(d / np.maximum(mag, rms)))


def phi_atom_err(p_gpu, p_ref):
    """max_i |dphi_i| / max(|phi_i|, rms phi)."""
    p_ref = np.asarray(p_ref, np.float64)
    d = np.abs(np.asarray(p_gpu, np.float64) - p_ref)
    rms = np.sqrt(np.mean(p_ref ** 2))
    return float(np.max(d / np.maximum(np.abs(p_ref), rms)))


def dvdl_ok(coul_gpu, coul_ref, term_mag, tol=RTOL):
    scale = np.maximum(np.abs(coul_ref), term_mag)
    err = np.abs(np.asarray(coul_gpu) - coul_ref) / scale
    return bool(np.all(err <= tol)), float(err.max()) if len(err) else 0.0


def energy_total(e):
    return sum(e[k] for k in POT_TERMS) + e["KE_atoms"] + e["KE_lambda"]


def compare_snapshot(ctx, r, ref, lam_atoms=None):
    """Compare a GPU context's replica r with an evaluated OracleReplica; returns dict of errors."""
    cur = ref.cur
    f, phi = ctx.cph_get_forces(r)
    coul, bias = ctx.cph_get_dvdl(r)
    e = ctx.cph_get_energies(r)
    eo = ref.energies()
    out = dict(force=force_err(f, cur["F"]), phi=phi_err(phi, cur["phi"]),
               force_atom=force_atom_err(f, cur["F"]), phi_atom=phi_atom_err(phi, cur["phi"]))
    ok, derr = dvdl_ok(coul, cur["dvdl_coul"], cur["term_mag"])
    out["dvdl_coul"] = derr
    out["dvdl_bias"] = float(np.max(np.abs(bias - cur["dvdl_bias"]) / np.maximum(1.0, np.abs(cur["dvdl_bias"])))) \
        if len(bias) else 0.0
    out["E_total"] = abs(e["total"] - eo["total"]) / abs(eo["total"])
    out["E_terms"] = {k: (e[k], eo[k]) for k in eo}
    if lam_atoms is not None and len(lam_atoms):
        rms = np.sqrt(np.mean(cur["phi"] ** 2))
        d = np.abs(phi[lam_atoms] - cur["phi"][lam_atoms]) / np.maximum(np.abs(cur["phi"][lam_atoms]), rms)
        out["phi_lambda_atoms"] = float(d.max())
    return out
