"""CPU: the sm_100a library builds, loads, and exports exactly what include/*.h
declares; host helpers agree across the three implementations; without a GPU
the product fails loudly (no CPU fallback)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path
import re
import subprocess

import numpy as np
import pytest

from paper_1610_07159_b200 import build, capi
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, level_dims

ROOT = build.ROOT


def declared(header: str) -> set[str]:
    txt = (ROOT / "include" / header).read_text()
    return set(re.findall(r"\b(hwf_[a-z0-9_]+)\s*\(", txt))


def exported(lib) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], check=True, capture_output=True, text=True).stdout
    return {l.split()[-1] for l in out.splitlines() if " T hwf_" in l}


@pytest.fixture(scope="module")
def cuda_lib():
    return build.build_cuda()


def test_cuda_library_exports_every_declared_symbol(cuda_lib):
    decl = declared("hwflow_c.h") | declared("hwflow_ext.h") | declared("hwflow_split.h")
    assert decl, "no declarations parsed"
    assert decl <= exported(cuda_lib), decl - exported(cuda_lib)
    assert set(capi.EXPORTED) == declared("hwflow_c.h")
    assert set(capi.EXPORTED_EXT) == declared("hwflow_ext.h")
    assert set(capi.EXPORTED_SPLIT) == declared("hwflow_split.h")


def test_oracle_libraries_export_the_reference_boundary():
    build.build_oracle()
    for lib in (build.ORACLE_LIB, build.REF_LIB):
        if lib.exists():
            assert declared("hwflow_c.h") | declared("hwflow_split.h") <= exported(lib)


def test_cuda_library_is_sm100a(cuda_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(cuda_lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_helpers_agree(cuda_lib):
    libs = [capi.Library(cuda_lib), capi.Library(build.ORACLE_LIB)]
    for w, h, L, step in ((640, 480, 4, 8), (1920, 1080, 5, 8), (3840, 2160, 5, 4), (40, 20, 5, 2), (7, 5, 3, 1)):
        dims = [level_dims(l, w, h, L, step) for l in libs]
        assert dims[0] == dims[1]
    assert level_dims(libs[0], 640, 480, 4, 8) == [(640, 480, 81, 61), (320, 240, 41, 31), (160, 120, 21, 16),
                                                   (80, 60, 11, 9)]
    for l in libs:
        for name in ("live", "facial", "stereo-hq"):
            p = capi.EnergyParamsC()
            assert l.hwf_preset_params(name.encode(), C.byref(p)) == capi.HWF_OK
            ref = EnergyParams.preset(name)
            assert [getattr(p, f) for f, _ in capi.EnergyParamsC._fields_] == [getattr(ref, f) for f, _ in
                                                                              capi.EnergyParamsC._fields_]
        assert l.hwf_preset_params(b"nope", C.byref(capi.EnergyParamsC())) == capi.HWF_EINVAL
        s = capi.ScheduleC()
        l.hwf_default_schedule(C.byref(s))
        d = SolveSchedule()
        assert (s.levels, s.pcg_iters, s.patch_iters, s.subdomain_px, s.boundary_px, s.grid_step) == (
            d.levels, d.pcg_iters, d.patch_iters, d.subdomain_px, d.boundary_px, d.grid_step)
        bad = EnergyParams(eps_huber=0.0).to_c()
        assert l.hwf_validate_params(C.byref(bad)) == capi.HWF_EINVAL


def test_product_has_no_cpu_fallback(cuda_lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = capi.Library(cuda_lib)
    h = C.c_void_p()
    assert lib.hwf_create(0, C.byref(h)) == capi.HWF_ECUDA
    from paper_1610_07159_b200.hwflow import Solver
    with pytest.raises(capi.HwflowError):
        Solver(cuda_lib)


def test_synthetic_pull_back_is_exact():
    from paper_1610_07159_b200 import synthetic
    T = synthetic.Texture(5, 64, 48)
    x = np.array([10.25, 30.5]), np.array([7.75, 20.0])
    a = synthetic.render_pair(64, 48, s=(1.5, 0.25), m=(0.5, -0.75), seed=5, noise=0.0, dtype=np.float64)
    # I_c^t(warp_position(x)) = T(x) at integer x where warp lands on integers
    s, m = (1.0, 0.0), (0.0, 0.0)
    b = synthetic.render_pair(64, 48, s=s, m=m, seed=5, noise=0.0, dtype=np.float64)
    assert np.allclose(b[1][:, 2:], b[0][:, :-2])  # right = left shifted by disparity 2 s_x
    assert a.shape == (4, 48, 64) and T(*x).shape == (2,)


def test_reference_side_bridge_compiles():
    """include/hwflow_bridge.hpp (the adapter a reference maintainer adds) compiles
    against the reference's own headers (with the Eigen shim)."""
    ref_inc = Path("/root/reference/proj/include")
    if not ref_inc.exists():
        pytest.skip("reference headers not present")
    src = "#include \"hwflow_bridge.hpp\"\nint main() { return 0; }\n"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-", f"-I{ROOT / 'include'}",
                        f"-I{ROOT / 'oracle' / 'eigen_shim'}", f"-I{ref_inc}"], input=src, capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr[-2000:]
