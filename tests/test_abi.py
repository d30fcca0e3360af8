"""CPU checks of the boundary: the C-ABI library loads and exports every symbol declared in
include/sph.h (no compute calls without a GPU); argument validation happens before device work."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2604_12505_b200 import build
    return build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "sph.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sph_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(libpath):
    names = _declared()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sph_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = C.CDLL(libpath)
    for n in names:
        assert getattr(L, n) is not None


def test_binding_covers_header(libpath):
    from paper_2604_12505_b200 import binding
    assert set(binding.exported_symbols()) == set(_declared())
    binding.lib()


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_80", "sm_90", "sm_89"):
        assert other + "." not in out


def test_invalid_parameters_rejected_without_gpu(libpath):
    """Config errors are reported before any device work (sph_workspace_bytes returns 0)."""
    import sph_inputs as si
    from paper_2604_12505_b200 import binding as B
    L = B.lib()
    sp = si.preset(1.0)
    fp, bp, tp = B.fluid_params(sp), B.body_params(sp), B.time_params(sp)
    ok = L.sph_workspace_bytes(C.byref(fp), C.byref(bp), C.byref(tp), 569, 236, 4)
    assert ok > 569 * 4 * 64
    for field, bad in (("h", 0.0), ("gamma1", 1.5), ("eps", 0.0), ("rho0", -1.0)):
        f2 = B.fluid_params(sp)
        setattr(f2, field, bad)
        assert L.sph_workspace_bytes(C.byref(f2), C.byref(bp), C.byref(tp), 569, 236, 4) == 0
    t2 = B.time_params(sp, rebin_every=0, skin=0.0)
    assert L.sph_workspace_bytes(C.byref(fp), C.byref(bp), C.byref(t2), 569, 236, 4) == 0
    assert L.sph_workspace_bytes(C.byref(fp), C.byref(bp), C.byref(tp), 569, 236, 0) == 0
    # init with a too-small workspace fails with ENOMEM before touching the device
    ctx = C.c_void_p()
    import numpy as np
    pv = np.zeros((569, 4), np.float32)
    gb = si.ghost_ring(236)
    st = L.sph_init_tank(C.byref(fp), C.byref(bp), C.byref(tp), 569, pv.ctypes.data, 236,
                         gb.ctypes.data, 1, None, 256, 1024, C.byref(ctx))
    assert st == B.SPH_ENOMEM
    assert b"workspace" in L.sph_last_error(None)
    # ghosts not on the wall circle are rejected
    st = L.sph_init_tank(C.byref(fp), C.byref(bp), C.byref(tp), 569, pv.ctypes.data, 236,
                         (gb * 0.9).ctypes.data, 1, None, 256, 1 << 40, C.byref(ctx))
    assert st == B.SPH_EINVAL


def test_null_context_calls_rejected_without_gpu(libpath):
    """Every entry point that takes a context returns SPH_EINVAL for a NULL context or NULL
    buffers before touching the device (header: 'Argument / configuration errors return
    SPH_EINVAL before any device work')."""
    from paper_2604_12505_b200 import binding as B
    L = B.lib()
    buf = (C.c_double * 64)()
    assert L.sph_jacobian(None, 0, buf, buf, 0) == B.SPH_EINVAL
    assert L.sph_eigenvalues(None, 4, buf, buf, 0) == B.SPH_EINVAL
    assert L.sph_step(None, None, 1, 0) == B.SPH_EINVAL
    assert L.sph_get_body_state(None, buf) == B.SPH_EINVAL
    assert L.sph_set_live_timing(None, 4) == B.SPH_EINVAL
    assert L.sph_get_live_timing(None, buf, None, 0) == B.SPH_EINVAL
    assert L.sph_settle(None, 0.5, 10) == B.SPH_EINVAL
    assert L.sph_launches_per_substep(None) == 0
