"""C-ABI library checks that need no GPU: it loads, exports every symbol include/cph.h
declares, and rejects invalid input before touching a device."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cph():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2410_01626_b200 as m
    return m


def test_every_header_symbol_is_exported(cph):
    hdr = open(os.path.join(ROOT, "include", "cph.h")).read()
    names = set(re.findall(r"\b(cph_[a-z_A-Z0-9]+)\s*\(", hdr))
    assert len(names) >= 20
    lib = cph.lib()
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert set(names) == set(cph.binding.EXPORTS)


def test_sm100a_code_in_library():
    import subprocess
    so = os.path.join(ROOT, "paper_2410_01626_b200", "libcph.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _sys():
    from synthetic.systems import small_system
    return small_system()


@pytest.mark.parametrize("mutate,msg", [
    (lambda s: s.pos.__setitem__((0, 0), np.nan), "non-finite"),
    (lambda s: s.state_q.__setitem__((0, slice(2, 4)), s.state_q[0, 2:4] + 0.1), "total charge"),
    (lambda s: s.group_kind.__setitem__(0, 4), "group_kind"),
    (lambda s: s.type.__setitem__(0, 99), "type out of range"),
    (lambda s: s.excl.__setitem__((0, 1), s.excl[0, 0]), "exclusion"),
])
def test_invalid_system_rejected(cph, mutate, msg):
    s = _sys()
    mutate(s)
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0], [1], use_torch_allocator=False)
    assert ei.value.status == 1 and msg in str(ei.value)


def test_invalid_params_rejected(cph):
    s = _sys()
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0], [1], rlist=1.2, use_torch_allocator=False)      # box 2.3 -> rlist >= L/2
    assert ei.value.status == 1
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0], [1], pme_order=6, use_torch_allocator=False)
    assert ei.value.status == 6
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0], [1], pme_grid=(22, 22, 22), use_torch_allocator=False)   # 11 not smooth
    assert ei.value.status == 6
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [np.nan], [1], use_torch_allocator=False)
    assert ei.value.status == 1


def test_dbo_defaults_are_the_papers(cph):
    """cph_default_params carries the DBO constants of PAPER.md:778-798 (off by default)."""
    import ctypes
    p = cph.binding.cph_params()
    cph.lib().cph_default_params(ctypes.byref(p))
    assert p.abi_version == 5 and p.deterministic == 0 and p.sub_batches == 0 and p.pair_list == 0 and p.dbo_well == 0 and p.dbo_barrier == 0
    assert (p.dbo_well_steps, p.dbo_barrier_steps, p.dbo_censor_steps) == (20000, 500000, 5000)   # 40 ps, 1 ns, 10 ps
    assert (p.dbo_well_near, p.dbo_residency, p.dbo_well_tol, p.dbo_well_gain, p.dbo_well_cap) == (0.2, 0.7, 0.03, 0.5, 0.08)
    assert (p.dbo_trans_lo, p.dbo_trans_hi, p.dbo_target, p.dbo_target_tol) == (0.2, 0.8, 0.25, 0.05)
    assert (p.dbo_barrier_step, p.dbo_barrier_min, p.dbo_barrier_max, p.barrier) == (1.0, 1.0, 20.0, 6.0)


def test_invalid_dbo_params_rejected(cph):
    s = _sys()
    for kw in (dict(dbo_well=1, dbo_well_steps=15),            # not a multiple of nstlist = 10
               dict(dbo_barrier=1, dbo_barrier_steps=0),
               dict(dbo_well=1, dbo_well_cap=0.5),
               dict(dbo_barrier=1, dbo_barrier_min=5.0, dbo_barrier_max=2.0)):
        with pytest.raises(cph.CphError) as ei:
            cph.cph_create(s, [4.0], [1], use_torch_allocator=False, **kw)
        assert ei.value.status == 1 and "DBO" in str(ei.value), kw


def test_unknown_override_rejected(cph):
    """SPEC.md:77 "unknown keys are errors": a misspelt parameter never silently falls back
    to its default."""
    s = _sys()
    with pytest.raises(ValueError, match="gama_atom"):
        cph.cph_create(s, [4.0], [1], gama_atom=3.0, use_torch_allocator=False)


@pytest.mark.parametrize("labels", [[0, 0, 1], [0, 2, 2], [1, 1, 1]])
def test_replica_exchange_ladders_must_be_permutations(cph, labels):
    """A ladder held by one context must carry every pH level exactly once (ADVICE r1:
    duplicate labels would corrupt the level assignment in k_remd_apply)."""
    s = _sys()
    levels = [4.0, 5.0, 6.0]
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [levels[k] for k in labels], [1, 2, 3], ph_levels=levels, use_torch_allocator=False)
    assert ei.value.status == 1 and "ladder" in str(ei.value)


def test_sub_batches_validated(cph):
    """cph_params.sub_batches: negative is an error; a pH ladder split across two replica
    sub-batches is checked as a whole by the context (each sub-batch sees only part of it)."""
    s = _sys()
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0], [1], sub_batches=-1, use_torch_allocator=False)
    assert ei.value.status == 1 and "sub_batches" in str(ei.value)
    levels = [4.0, 5.0]
    # R = 4 in 3 sub-batches (2, 1, 1): ladder 1 = replicas 2, 3 spans batches 1 and 2
    with pytest.raises(cph.CphError) as ei:
        cph.cph_create(s, [4.0, 5.0, 5.0, 5.0], [1, 2, 3, 4], ph_levels=levels, sub_batches=3,
                       use_torch_allocator=False)
    assert ei.value.status == 1 and "ladder" in str(ei.value)
