"""ctypes binding of include/cph.h: argument marshalling only.

Every step of the computation runs in libcph.so's CUDA kernels; this module only
converts numpy arrays to pointers, keeps them alive for the duration of the
call, and raises on a non-zero cph_status.  There is no CPU fallback: if the
shared library is missing or cannot be loaded, importing the package raises.
PyTorch (optional) supplies device memory (its caching allocator) and the
CUDA stream, per the north star's "PyTorch only for memory, streams and
process groups".
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPH_LIB", os.path.join(_HERE, "libcph.so"))   # CPH_LIB: A/B builds

CPH_ABI_VERSION = 5
STATUS = {0: "CPH_OK", 1: "CPH_E_INVALID", 2: "CPH_E_CUDA", 3: "CPH_E_DIVERGED", 4: "CPH_E_STATE",
          5: "CPH_E_OOM", 6: "CPH_E_UNSUPPORTED"}
ENERGY_TERMS = ("LJ", "real", "excl", "self", "recip", "net", "hi", "bias", "KE_atoms", "KE_lambda", "total")
KERNEL_CLASSES = ("integrate", "pairlist", "nonbonded", "spread", "fft_r2c", "solve", "fft_c2r",
                  "gather", "lambda", "hi")
N_ETERMS = len(ENERGY_TERMS)

_p = C.POINTER
_f32p, _f64p, _i32p, _u64p, _i64p = _p(C.c_float), _p(C.c_double), _p(C.c_int32), _p(C.c_uint64), _p(C.c_int64)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class cph_system(C.Structure):
    _fields_ = [("n_atoms", C.c_int32), ("pos", _f32p), ("vel", _f32p), ("mass", _f32p), ("charge", _f32p),
                ("type", _i32p), ("n_types", C.c_int32), ("c6", _f64p), ("c12", _f64p),
                ("n_excl", C.c_int32), ("excl", _i32p), ("box", C.c_double * 3), ("n_groups", C.c_int32),
                ("group_kind", _i32p), ("group_ptr", _i32p), ("group_atoms", _i32p), ("state_q", _f64p),
                ("is_buffer", _i32p), ("pKa", _f64p), ("vmm", _f64p)]


class cph_params(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("n_replicas", C.c_int32), ("device", C.c_int32), ("mode", C.c_int32),
                ("dt", C.c_double), ("temperature", C.c_double), ("gamma_atom", C.c_double),
                ("gamma_lambda", C.c_double), ("lambda_mass", C.c_double), ("rc", C.c_double),
                ("rlist", C.c_double), ("ewald_rtol", C.c_double), ("pme_grid", C.c_int32 * 3),
                ("pme_order", C.c_int32), ("nstlist", C.c_int32), ("nstout", C.c_int32), ("nstenergy", C.c_int32),
                ("barrier", C.c_double), ("wall_k", C.c_double), ("pH", _f64p), ("replica_seed", _u64p),
                ("lambda0", _f64p), ("pos_replicas", _f32p), ("vel_replicas", _f32p),
                ("frame_capacity", C.c_int32), ("cuda_stream", C.c_void_p), ("dev_alloc", ALLOC_FN),
                ("dev_free", FREE_FN), ("alloc_ctx", C.c_void_p),
                ("dbo_well", C.c_int32), ("dbo_barrier", C.c_int32), ("dbo_well_steps", C.c_int64),
                ("dbo_barrier_steps", C.c_int64), ("dbo_censor_steps", C.c_int64), ("dbo_well_near", C.c_double),
                ("dbo_residency", C.c_double), ("dbo_well_tol", C.c_double), ("dbo_well_gain", C.c_double),
                ("dbo_well_cap", C.c_double), ("dbo_trans_lo", C.c_double), ("dbo_trans_hi", C.c_double),
                ("dbo_target", C.c_double), ("dbo_target_tol", C.c_double), ("dbo_barrier_step", C.c_double),
                ("dbo_barrier_min", C.c_double), ("dbo_barrier_max", C.c_double),
                ("thermostat", C.c_int32), ("tau_atom", C.c_double), ("tau_lambda", C.c_double),
                ("n_ph_levels", C.c_int32), ("ph_levels", _f64p), ("remd_first", C.c_int32),
                ("remd_total", C.c_int32), ("hamiltonian", C.c_int32), ("deterministic", C.c_int32),
                ("sub_batches", C.c_int32), ("pair_list", C.c_int32)]


class cph_dbo_event(C.Structure):
    _fields_ = [("step", C.c_int64), ("replica", C.c_int32), ("coord", C.c_int32), ("kind", C.c_int32),
                ("pad", C.c_int32), ("old_value", C.c_double), ("new_value", C.c_double)]


DBO_KINDS = ("well0", "well1", "barrier", "barrier_t_prot", "barrier_t_deprot")


EXPORTS = {
    "cph_default_params": (None, [_p(cph_params)]),
    "cph_create": (C.c_int, [_p(cph_system), _p(cph_params), _p(C.c_void_p)]),
    "cph_destroy": (None, [C.c_void_p]),
    "cph_get_stream": (C.c_void_p, [C.c_void_p]),
    "cph_n_coords": (C.c_int32, [C.c_void_p]),
    "cph_n_atoms": (C.c_int32, [C.c_void_p]),
    "cph_n_replicas": (C.c_int32, [C.c_void_p]),
    "cph_n_sub_batches": (C.c_int32, [C.c_void_p]),
    "cph_set_pH": (C.c_int, [C.c_void_p, C.c_int32, C.c_double]),
    "cph_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "cph_sync": (C.c_int, [C.c_void_p]),
    "cph_current_step": (C.c_int64, [C.c_void_p]),
    "cph_get_lambdas": (C.c_int, [C.c_void_p, C.c_int32, _f64p, _f64p]),
    "cph_get_dvdl": (C.c_int, [C.c_void_p, C.c_int32, _f64p, _f64p]),
    "cph_get_energies": (C.c_int, [C.c_void_p, C.c_int32, _f64p]),
    "cph_get_bias_params": (C.c_int, [C.c_void_p, C.c_int32, _f64p]),
    "cph_get_frames": (C.c_int, [C.c_void_p, C.c_int32, _f32p, C.c_int64, _i64p, _i64p]),
    "cph_get_frames_ex": (C.c_int, [C.c_void_p, C.c_int32, _f32p, _p(C.c_uint8), _i64p, _i32p, C.c_int64, _i64p,
                                    _i64p]),
    "cph_exchange_energies": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cph_exchange_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64]),
    "cph_exchange": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64]),
    "cph_get_labels": (C.c_int, [C.c_void_p, _i32p]),
    "cph_set_labels": (C.c_int, [C.c_void_p, _i32p]),
    "cph_get_exchange_stats": (C.c_int, [C.c_void_p, _i64p, _i64p]),
    "cph_get_dbo_params": (C.c_int, [C.c_void_p, C.c_int32, _f64p]),
    "cph_set_dbo_params": (C.c_int, [C.c_void_p, C.c_int32, _f64p]),
    "cph_get_dbo_events": (C.c_int, [C.c_void_p, _p(cph_dbo_event), C.c_int64, _i64p]),
    "cph_get_dbo_stats": (C.c_int, [C.c_void_p, C.c_int32, _f64p, _f64p]),
    "cph_get_forces": (C.c_int, [C.c_void_p, C.c_int32, _f32p, _f32p]),
    "cph_get_positions": (C.c_int, [C.c_void_p, C.c_int32, _f32p, _f32p]),
    "cph_get_pairlist": (C.c_int, [C.c_void_p, C.c_int32, _i32p, C.c_int64, _i64p]),
    "cph_get_pairlist_directed": (C.c_int, [C.c_void_p, C.c_int32, _i32p, C.c_int64, _i64p]),
    "cph_get_lambda_groups": (C.c_int, [C.c_void_p, C.c_int32, _i32p, _i32p, _i32p, _i32p]),
    "cph_get_pairlist_rows": (C.c_int, [C.c_void_p, C.c_int32, _i32p, C.c_int32, _i32p, _i32p, C.c_int64]),
    "cph_get_ti_means": (C.c_int, [C.c_void_p, C.c_int32, _f64p, _i64p]),
    "cph_get_state": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, _i64p]),
    "cph_set_state": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]),
    "cph_get_state_all": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, _i64p]),
    "cph_set_state_all": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "cph_profile_steps": (C.c_int, [C.c_void_p, C.c_int64, _f64p, _i64p]),
    "cph_launch_count": (C.c_int64, [C.c_void_p]),
    "cph_last_error": (C.c_char_p, [C.c_void_p]),
}


class CphError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def load_library(path: str = LIB_PATH):
    """Load libcph.so and declare every exported symbol; raises if anything is missing."""
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c \"import __graft_entry__ as g; g.build()\"` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def _ptr(a, ctype):
    return a.ctypes.data_as(_p(ctype)) if a is not None else None


def _check(st, ctx=None):
    if st != 0:
        raise CphError(st, (lib().cph_last_error(ctx) or b"").decode())


def _torch_allocator(device):
    import torch

    def alloc(nbytes, _ctx):
        return torch.cuda.caching_allocator_alloc(int(nbytes), device=device)

    def free(ptr, _ctx):
        try:
            torch.cuda.caching_allocator_delete(ptr)
        except Exception:          # interpreter shutdown: torch may already be torn down
            pass
    return ALLOC_FN(alloc), FREE_FN(free)


_FLOAT_PARAMS = ("dt", "temperature", "gamma_atom", "gamma_lambda", "lambda_mass", "rc", "rlist", "ewald_rtol",
                 "barrier", "wall_k", "tau_atom", "tau_lambda", "dbo_well_near", "dbo_residency", "dbo_well_tol",
                 "dbo_well_gain", "dbo_well_cap", "dbo_trans_lo", "dbo_trans_hi", "dbo_target", "dbo_target_tol",
                 "dbo_barrier_step", "dbo_barrier_min", "dbo_barrier_max")
_INT_PARAMS = ("pme_order", "nstlist", "nstout", "nstenergy", "frame_capacity", "dbo_well", "dbo_barrier",
               "dbo_well_steps", "dbo_barrier_steps", "dbo_censor_steps", "hamiltonian", "deterministic",
               "sub_batches", "pair_list")
KNOWN_PARAMS = frozenset(_FLOAT_PARAMS + _INT_PARAMS + ("thermostat", "pme_grid"))


def cph_create(system, pH, replica_seed, *, lambda0=None, pos_replicas=None, vel_replicas=None, device=0,
               mode=0, cuda_stream=None, use_torch_allocator=True, ph_levels=None, remd_first=0, remd_total=0,
               **overrides):
    """Create a context for R = len(pH) replicas of `system` (any object with the
    SyntheticSystem attributes).  Parameter overrides use cph_params field names.
    ph_levels (sorted pH values) enables pH replica exchange."""
    L = lib()
    pH = np.ascontiguousarray(pH, np.float64).reshape(-1)
    R = len(pH)
    seeds = np.ascontiguousarray(replica_seed, np.uint64).reshape(-1)
    if len(seeds) != R:
        raise ValueError("need one seed per replica")
    keep = []

    def arr(x, dt):
        if x is None:
            return None
        a = np.ascontiguousarray(x, dt)
        keep.append(a)
        return a
    s = cph_system()
    pos = arr(system.pos, np.float32)
    s.n_atoms = pos.shape[0]
    s.pos = _ptr(pos, C.c_float)
    s.vel = _ptr(arr(getattr(system, "vel", None), np.float32), C.c_float)
    s.mass = _ptr(arr(system.mass, np.float32), C.c_float)
    s.charge = _ptr(arr(system.charge, np.float32), C.c_float)
    s.type = _ptr(arr(system.type, np.int32), C.c_int32)
    c6 = arr(system.c6, np.float64)
    s.n_types = c6.shape[0]
    s.c6 = _ptr(c6, C.c_double)
    s.c12 = _ptr(arr(system.c12, np.float64), C.c_double)
    ex = arr(np.asarray(system.excl).reshape(-1, 2), np.int32)
    s.n_excl = ex.shape[0]
    s.excl = _ptr(ex, C.c_int32)
    s.box[:] = [float(b) for b in system.box]
    gk = arr(system.group_kind, np.int32)
    s.n_groups = gk.shape[0]
    s.group_kind = _ptr(gk, C.c_int32)
    s.group_ptr = _ptr(arr(system.group_ptr, np.int32), C.c_int32)
    s.group_atoms = _ptr(arr(system.group_atoms, np.int32), C.c_int32)
    s.state_q = _ptr(arr(system.state_q, np.float64), C.c_double)
    s.is_buffer = _ptr(arr(system.is_buffer, np.int32), C.c_int32)
    s.pKa = _ptr(arr(system.pKa, np.float64), C.c_double)
    s.vmm = _ptr(arr(system.vmm, np.float64), C.c_double)

    p = cph_params()
    L.cph_default_params(C.byref(p))
    p.n_replicas = R
    p.device = device
    p.mode = mode
    unknown = sorted(set(overrides) - KNOWN_PARAMS)
    if unknown:                     # SPEC.md:77 "unknown keys are errors"
        raise ValueError(f"unknown cph_params override(s): {', '.join(unknown)}")
    params = dict(getattr(system, "params", {}))
    params.update(overrides)
    for k in _FLOAT_PARAMS:
        if k in params:
            setattr(p, k, float(params[k]))
    for k in _INT_PARAMS:
        if k in params:
            setattr(p, k, int(params[k]))
    if "thermostat" in params:
        t = params["thermostat"]
        p.thermostat = {"langevin": 0, "bussi": 1}[t] if isinstance(t, str) else int(t)
    grid = overrides.get("pme_grid", getattr(system, "pme_grid", None))
    if grid is not None:
        p.pme_grid[:] = [int(g) for g in grid]
    p.pH = _ptr(arr(pH, np.float64), C.c_double)
    p.replica_seed = _ptr(arr(seeds, np.uint64), C.c_uint64)
    p.lambda0 = _ptr(arr(lambda0, np.float64), C.c_double)
    p.pos_replicas = _ptr(arr(pos_replicas, np.float32), C.c_float)
    p.vel_replicas = _ptr(arr(vel_replicas, np.float32), C.c_float)
    if ph_levels is not None:
        lv = arr(ph_levels, np.float64).reshape(-1)
        p.n_ph_levels = len(lv)
        p.ph_levels = _ptr(lv, C.c_double)
        p.remd_first = int(remd_first)
        p.remd_total = int(remd_total)
    p.cuda_stream = cuda_stream
    cbs = None
    if use_torch_allocator:
        try:
            import torch
            if torch.cuda.is_available():
                cbs = _torch_allocator(device)
                p.dev_alloc, p.dev_free = cbs
                if cuda_stream is None:
                    # torch's legacy default stream has handle 0; the library then uses its own
                    # stream (graph capture is not allowed on the legacy stream)
                    p.cuda_stream = torch.cuda.current_stream(device).cuda_stream or None
        except ImportError:
            cbs = None
    h = C.c_void_p()
    _check(L.cph_create(C.byref(s), C.byref(p), C.byref(h)))
    return Context(h, R, cbs, p.n_ph_levels, device)


class Context:
    """Owns a cph_ctx handle; methods are the cph_* getters with numpy outputs."""

    def __init__(self, handle, R, callbacks, n_levels=0, device=0):
        self.h = handle
        self.R = R
        self.P = n_levels
        self.device = device
        self._cbs = callbacks            # keep allocator callbacks alive
        self.C = lib().cph_n_coords(handle)
        self.N = lib().cph_n_atoms(handle)
        self.sub_batches = lib().cph_n_sub_batches(handle)

    def close(self):
        if self.h:
            lib().cph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def cph_step(self, n):
        _check(lib().cph_step(self.h, int(n)), self.h)

    def cph_sync(self):
        _check(lib().cph_sync(self.h), self.h)

    def cph_set_pH(self, r, pH):
        _check(lib().cph_set_pH(self.h, int(r), float(pH)), self.h)

    def cph_current_step(self):
        return int(lib().cph_current_step(self.h))

    def cph_launch_count(self):
        return int(lib().cph_launch_count(self.h))

    def cph_get_lambdas(self, r):
        lam = np.zeros(self.C)
        vel = np.zeros(self.C)
        _check(lib().cph_get_lambdas(self.h, r, _ptr(lam, C.c_double), _ptr(vel, C.c_double)), self.h)
        return lam, vel

    def cph_get_dvdl(self, r):
        a = np.zeros(self.C)
        b = np.zeros(self.C)
        _check(lib().cph_get_dvdl(self.h, r, _ptr(a, C.c_double), _ptr(b, C.c_double)), self.h)
        return a, b

    def cph_get_energies(self, r):
        e = np.zeros(N_ETERMS)
        _check(lib().cph_get_energies(self.h, r, _ptr(e, C.c_double)), self.h)
        return dict(zip(ENERGY_TERMS, e.tolist()))

    def cph_get_bias_params(self, r):
        d1 = np.zeros(self.C)
        _check(lib().cph_get_bias_params(self.h, r, _ptr(d1, C.c_double)), self.h)
        return d1

    def cph_get_frames(self, r, cap=1 << 20):
        cap = int(cap)
        buf = np.zeros(max(cap, 1) * max(self.C, 1), np.float32)
        n, dropped = C.c_int64(), C.c_int64()
        _check(lib().cph_get_frames(self.h, r, _ptr(buf, C.c_float), cap, C.byref(n), C.byref(dropped)), self.h)
        return buf[: n.value * self.C].reshape(n.value, self.C), dropped.value

    def cph_get_frames_ex(self, r, cap=1 << 20):
        """(frames [n, C], censored [n, C] bool, steps [n], pH-level labels [n], n_dropped)."""
        cap = int(cap)
        buf = np.zeros(max(cap, 1) * max(self.C, 1), np.float32)
        cen = np.zeros(max(cap, 1) * max(self.C, 1), np.uint8)
        st = np.zeros(max(cap, 1), np.int64)
        lab = np.zeros(max(cap, 1), np.int32)
        n, dropped = C.c_int64(), C.c_int64()
        _check(lib().cph_get_frames_ex(self.h, r, _ptr(buf, C.c_float), _ptr(cen, C.c_uint8), _ptr(st, C.c_int64),
                                       _ptr(lab, C.c_int32), cap, C.byref(n), C.byref(dropped)), self.h)
        k = n.value
        return (buf[: k * self.C].reshape(k, self.C), cen[: k * self.C].reshape(k, self.C).astype(bool),
                st[:k].copy(), lab[:k].copy(), dropped.value)

    # -- pH replica exchange -------------------------------------------------------------
    def cph_exchange_energies(self, rows_dev_ptr):
        _check(lib().cph_exchange_energies(self.h, C.c_void_p(int(rows_dev_ptr))), self.h)

    def cph_exchange_apply(self, rows_all_dev_ptr, seed, attempt):
        _check(lib().cph_exchange_apply(self.h, C.c_void_p(int(rows_all_dev_ptr)), int(seed), int(attempt)), self.h)

    def cph_exchange(self, seed, attempt):
        _check(lib().cph_exchange(self.h, int(seed), int(attempt)), self.h)

    def exchange_device(self):
        import torch
        return torch.device("cuda", self.device)

    def lib_stream(self):
        """The context's CUDA stream as a torch stream object (cph_get_stream)."""
        import torch
        return torch.cuda.ExternalStream(int(lib().cph_get_stream(self.h) or 0), device=self.exchange_device())

    def exchange_energies_into(self, t):
        """Write this context's (label, E_p) rows into the float64 CUDA tensor t.  Ordered
        after torch's current stream (which allocated / last used t) and before it (which
        runs the NCCL gather): the library writes on its own stream."""
        import torch
        assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() >= self.R * (self.P + 1)
        cur, ls = torch.cuda.current_stream(t.device), self.lib_stream()
        ls.wait_stream(cur)
        self.cph_exchange_energies(t.data_ptr())
        cur.wait_stream(ls)      # later use or reuse of t on torch's stream follows the write

    def exchange_apply_from(self, t, seed, attempt):
        """Apply the decisions from the gathered rows t (filled on torch's current stream)."""
        import torch
        assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
        cur, ls = torch.cuda.current_stream(t.device), self.lib_stream()
        ls.wait_stream(cur)
        self.cph_exchange_apply(t.data_ptr(), seed, attempt)
        cur.wait_stream(ls)      # the caching allocator may reuse t only after this read

    def cph_get_labels(self):
        lab = np.zeros(self.R, np.int32)
        _check(lib().cph_get_labels(self.h, _ptr(lab, C.c_int32)), self.h)
        return lab

    def cph_set_labels(self, labels):
        lab = np.ascontiguousarray(labels, np.int32)
        _check(lib().cph_set_labels(self.h, _ptr(lab, C.c_int32)), self.h)

    def cph_get_exchange_stats(self, n_ladders):
        n = n_ladders * (self.P - 1)
        a = np.zeros(max(n, 1), np.int64)
        b = np.zeros(max(n, 1), np.int64)
        _check(lib().cph_get_exchange_stats(self.h, _ptr(a, C.c_int64), _ptr(b, C.c_int64)), self.h)
        return a[:n].reshape(n_ladders, -1), b[:n].reshape(n_ladders, -1)

    def cph_get_dbo_params(self, r):
        """[C, 4]: (a0, a1, h_prot, h_deprot) per coordinate."""
        p = np.zeros(4 * self.C)
        _check(lib().cph_get_dbo_params(self.h, r, _ptr(p, C.c_double)), self.h)
        return p.reshape(self.C, 4)

    def cph_set_dbo_params(self, r, params):
        p = np.ascontiguousarray(params, np.float64).reshape(-1)
        _check(lib().cph_set_dbo_params(self.h, r, _ptr(p, C.c_double)), self.h)

    def cph_get_dbo_events(self, cap=4096):
        """Drained adjustment log: list of (step, replica, coord, kind name, old, new)."""
        out = []
        buf = (cph_dbo_event * cap)()
        n = C.c_int64()
        while True:
            _check(lib().cph_get_dbo_events(self.h, buf, cap, C.byref(n)), self.h)
            out += [(e.step, e.replica, e.coord, DBO_KINDS[e.kind], e.old_value, e.new_value) for e in buf[: n.value]]
            if n.value < cap:
                return out

    def cph_get_dbo_stats(self, r):
        w = np.zeros(5 * self.C)
        b = np.zeros(4 * self.C)
        _check(lib().cph_get_dbo_stats(self.h, r, _ptr(w, C.c_double), _ptr(b, C.c_double)), self.h)
        return w.reshape(self.C, 5), b.reshape(self.C, 4)

    def cph_get_forces(self, r):
        f = np.zeros((self.N, 3), np.float32)
        phi = np.zeros(self.N, np.float32)
        _check(lib().cph_get_forces(self.h, r, _ptr(f, C.c_float), _ptr(phi, C.c_float)), self.h)
        return f, phi

    def cph_get_positions(self, r):
        x = np.zeros((self.N, 3), np.float32)
        v = np.zeros((self.N, 3), np.float32)
        _check(lib().cph_get_positions(self.h, r, _ptr(x, C.c_float), _ptr(v, C.c_float)), self.h)
        return x, v

    def cph_get_pairlist(self, r):
        n = C.c_int64()
        _check(lib().cph_get_pairlist(self.h, r, None, 0, C.byref(n)), self.h)
        out = np.zeros(2 * max(n.value, 1), np.int32)
        _check(lib().cph_get_pairlist(self.h, r, _ptr(out, C.c_int32), n.value, C.byref(n)), self.h)
        return out[: 2 * n.value].reshape(-1, 2)

    def cph_get_pairlist_directed(self, r):
        n = C.c_int64()
        _check(lib().cph_get_pairlist_directed(self.h, r, None, 0, C.byref(n)), self.h)
        out = np.zeros(2 * max(n.value, 1), np.int32)
        _check(lib().cph_get_pairlist_directed(self.h, r, _ptr(out, C.c_int32), n.value, C.byref(n)), self.h)
        return out[: 2 * n.value].reshape(-1, 2)

    def cph_get_pairlist_rows(self, r, atoms):
        """List of sorted partner arrays (original indices) for each original atom index."""
        a = np.ascontiguousarray(atoms, np.int32)
        ptr = np.zeros(len(a) + 1, np.int32)
        _check(lib().cph_get_pairlist_rows(self.h, r, _ptr(a, C.c_int32), len(a), _ptr(ptr, C.c_int32), None, 0),
               self.h)
        cols = np.zeros(max(int(ptr[-1]), 1), np.int32)
        _check(lib().cph_get_pairlist_rows(self.h, r, _ptr(a, C.c_int32), len(a), _ptr(ptr, C.c_int32),
                                           _ptr(cols, C.c_int32), int(ptr[-1])), self.h)
        return [cols[ptr[k]:ptr[k + 1]].copy() for k in range(len(a))]

    def cph_get_lambda_groups(self, r, n_groups, n_lambda):
        """(group_ptr, coord_ptr, atoms via iperm, atoms via meta) as stored on the device."""
        gp = np.zeros(n_groups + 1, np.int32)
        cp = np.zeros(n_groups + 1, np.int32)
        a = np.zeros(max(n_lambda, 1), np.int32)
        b = np.zeros(max(n_lambda, 1), np.int32)
        _check(lib().cph_get_lambda_groups(self.h, r, _ptr(gp, C.c_int32), _ptr(cp, C.c_int32), _ptr(a, C.c_int32),
                                           _ptr(b, C.c_int32)), self.h)
        return gp, cp, a[:n_lambda], b[:n_lambda]

    def cph_get_ti_means(self, r):
        m = np.zeros(self.C)
        n = C.c_int64()
        _check(lib().cph_get_ti_means(self.h, r, _ptr(m, C.c_double), C.byref(n)), self.h)
        return m, n.value

    def cph_get_state(self, r):
        n = C.c_int64()
        _check(lib().cph_get_state(self.h, r, None, 0, C.byref(n)), self.h)
        buf = np.zeros(n.value, np.uint8)
        _check(lib().cph_get_state(self.h, r, buf.ctypes.data_as(C.c_void_p), n.value, C.byref(n)), self.h)
        return buf

    def cph_set_state(self, r, blob):
        blob = np.ascontiguousarray(blob, np.uint8)
        _check(lib().cph_set_state(self.h, r, blob.ctypes.data_as(C.c_void_p), blob.size), self.h)

    def cph_get_state_all(self, out=None):
        n = C.c_int64()
        _check(lib().cph_get_state_all(self.h, None, 0, C.byref(n)), self.h)
        buf = np.zeros(n.value, np.uint8) if out is None else out
        _check(lib().cph_get_state_all(self.h, buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(n)), self.h)
        return buf

    def cph_set_state_all(self, blob):
        blob = np.ascontiguousarray(blob, np.uint8)
        _check(lib().cph_set_state_all(self.h, blob.ctypes.data_as(C.c_void_p), blob.size), self.h)

    def cph_profile_steps(self, n):
        ms = np.zeros(len(KERNEL_CLASSES))
        cnt = np.zeros(len(KERNEL_CLASSES), np.int64)
        _check(lib().cph_profile_steps(self.h, int(n), _ptr(ms, C.c_double), _ptr(cnt, C.c_int64)), self.h)
        return dict(zip(KERNEL_CLASSES, ms.tolist())), dict(zip(KERNEL_CLASSES, cnt.tolist()))
