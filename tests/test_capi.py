"""C-ABI library: loads, exports every symbol include/dg.h declares, reports errors loudly (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1812_08075_b200 import build, dg
    build.build()
    return dg.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "dg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|double|const char\*)\s+(dg_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 14
    so = os.path.join(ROOT, "paper_1812_08075_b200", "lib", "libdg.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)
    from paper_1812_08075_b200 import dg
    assert set(dg.EXPORTS) == set(names)


def test_kernels_are_sm100a(lib):
    so = os.path.join(ROOT, "paper_1812_08075_b200", "lib", "libdg.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_without_device_or_bad_args(lib):
    from paper_1812_08075_b200 import dg
    import torch
    # NULL arguments are rejected before any CUDA call
    assert lib.dg_setup(None, 1, 2, None) == dg.DG_ERR_INVALID
    assert "NULL" in dg.dg_last_error()
    m = dg.dg_mesh()
    m.N[0] = m.N[1] = m.N[2] = 4
    m.nplanes = 4
    m.penalty_scale = 10.0
    h = ctypes.c_void_p()
    assert lib.dg_setup(ctypes.byref(m), 9, 10, ctypes.byref(h)) == dg.DG_ERR_INVALID
    assert lib.dg_setup(ctypes.byref(m), 2, 6, ctypes.byref(h)) == dg.DG_ERR_UNSUPPORTED  # k+4 points
    m.N[1] = 1
    assert lib.dg_setup(ctypes.byref(m), 2, 3, ctypes.byref(h)) == dg.DG_ERR_INVALID
    m.N[1] = 4
    m.geom_kind = 1  # affine without jac
    assert lib.dg_setup(ctypes.byref(m), 2, 3, ctypes.byref(h)) == dg.DG_ERR_INVALID
    m.geom_kind = 0
    if not torch.cuda.is_available():
        # no silent CPU path: a valid request fails loudly without a device
        with pytest.raises(dg.DgError) as ei:
            dg.dg_setup((4, 4, 4), 2, 3)
        assert ei.value.code == dg.DG_ERR_CUDA
    assert lib.dg_apply(None, None, None) == dg.DG_ERR_INVALID
    assert lib.dg_destroy(None) == dg.DG_OK


def test_problem_validation(lib):
    """The problem field: unknown kinds are invalid; the diffusion-reaction, nonlinear and Stokes problems are
    restricted to the combinations their kernels implement (DG_ERR_UNSUPPORTED otherwise), checked before any
    CUDA call; the Jacobian entry rejects NULL arguments."""
    from paper_1812_08075_b200 import dg
    m = dg.dg_mesh()
    m.N[0] = m.N[1] = m.N[2] = 4
    m.nplanes = 4
    m.penalty_scale = 3.0
    h = ctypes.c_void_p()
    m.problem = 7
    assert lib.dg_setup(ctypes.byref(m), 2, 4, ctypes.byref(h)) == dg.DG_ERR_INVALID
    for prob in (dg.DG_PROBLEM_DIFFREAC, dg.DG_PROBLEM_NLREAC):
        m.problem = prob
        assert lib.dg_setup(ctypes.byref(m), 2, 3, ctypes.byref(h)) == dg.DG_ERR_UNSUPPORTED  # needs quad = k+2
        m.coeff_kind = dg.DG_COEFF_SINCOS
        assert lib.dg_setup(ctypes.byref(m), 2, 4, ctypes.byref(h)) == dg.DG_ERR_UNSUPPORTED
        m.coeff_kind = dg.DG_COEFF_ONE
    m.problem = dg.DG_PROBLEM_STOKES
    assert lib.dg_setup(ctypes.byref(m), 2, 4, ctypes.byref(h)) == dg.DG_ERR_UNSUPPORTED  # needs quad = k+1
    assert "Stokes" in dg.dg_last_error()
    assert lib.dg_apply_jacobian(None, None, None, None) == dg.DG_ERR_INVALID
    assert lib.dg_apply_jacobian_planes(None, None, None, None, None, None, 0, 0) == dg.DG_ERR_INVALID


def test_slab_range_matches_slab_plan(lib):
    """dg_slab_range (the collective form's partition, host-only) == slab.plan (the torch.distributed form)."""
    from paper_1812_08075_b200 import dg, slab
    for N0 in (2, 5, 96, 256):
        for P in (1, 2, 3, 4, 8):
            if N0 < P:
                with pytest.raises(dg.DgError):
                    dg.dg_slab_range(N0, 0, P)
                continue
            for q in range(P):
                p = slab.plan(N0, q, P)
                assert dg.dg_slab_range(N0, q, P) == (p.plane_begin, p.nplanes)


def test_setup_dist_rejects_bad_args(lib):
    from paper_1812_08075_b200 import dg
    m = dg.dg_mesh()
    m.N[0] = m.N[1] = m.N[2] = 4
    m.nplanes = 4
    m.penalty_scale = 10.0
    h = ctypes.c_void_p()
    idb = ctypes.create_string_buffer(128)
    assert lib.dg_setup_dist(ctypes.byref(m), 2, 3, 0, 2, None, ctypes.byref(h)) == dg.DG_ERR_INVALID  # no id
    assert lib.dg_setup_dist(ctypes.byref(m), 2, 3, 2, 2, idb, ctypes.byref(h)) == dg.DG_ERR_INVALID    # rank
    assert lib.dg_setup_dist(ctypes.byref(m), 2, 3, 0, 2, idb, ctypes.byref(h)) == dg.DG_ERR_INVALID    # slab != rank 0's
    assert "slab" in dg.dg_last_error()
    assert lib.dg_apply_dist(None, None, None) == dg.DG_ERR_INVALID
