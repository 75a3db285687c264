"""CPU checks of the boundary: the C-ABI library builds, loads, exports every
symbol include/gscache.h declares, and rejects bad arguments without a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gsclib():
    import paper_2502_14938_b200 as p
    p.build()
    return p._abi


def _declared():
    txt = open(os.path.join(ROOT, "include", "gscache.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gsc_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("gsc_create", "gsc_load_scene", "gsc_set_pose", "gsc_render_pair", "gsc_destroy"):
        assert must in names


def test_every_declared_symbol_is_exported(gsclib):
    L = C.CDLL(gsclib.SO_PATH)
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(gsclib._SIGS)   # the binding covers exactly the header


def test_abi_version_and_argument_checks(gsclib):
    L = gsclib.lib()
    assert L.gsc_abi_version() == 4
    h = C.c_void_p()
    cfg = gsclib.gsc_config()
    assert L.gsc_create(0, C.byref(cfg), C.byref(h)) == gsclib.GSC_EINVAL      # zero-sized image
    cfg.width, cfg.height, cfg.fov_y, cfg.near_plane, cfg.far_plane, cfg.d_max = 64, 64, 1.2, 0.05, 100.0, 10
    cfg.near_plane = 200.0
    assert L.gsc_create(0, C.byref(cfg), C.byref(h)) == gsclib.GSC_EINVAL      # near >= far
    cfg.near_plane = 0.05
    cfg.fov_y = 3.2
    assert L.gsc_create(0, C.byref(cfg), C.byref(h)) == gsclib.GSC_EINVAL      # fov >= pi
    assert L.gsc_render_pair(None, None, None, 0, None, None) == gsclib.GSC_EINVAL
    assert L.gsc_last_error(None) == b"null context"


def test_no_gpu_means_loud_failure(gsclib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = gsclib.lib()
    h = C.c_void_p()
    cfg = gsclib.gsc_config()
    cfg.width, cfg.height, cfg.fov_y, cfg.near_plane, cfg.far_plane, cfg.d_max = 64, 64, 1.2, 0.05, 100.0, 10
    assert L.gsc_create(0, C.byref(cfg), C.byref(h)) == gsclib.GSC_ECUDA


def test_bounds_checked_debug_build_compiles_its_checks(gsclib):
    """tools/bounds_build.py (the stand-in for compute-sanitizer memcheck) still builds, its library
    carries the GSC_CHECK trap sites, and the product library does not (the checks compile away)."""
    import shutil
    import subprocess
    import sys
    if not shutil.which("cuobjdump") and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("no cuobjdump")
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bounds_build.py")], capture_output=True,
                         text=True, check=True).stdout.strip().splitlines()[-1]
    assert out.endswith("libgscache.so") and os.path.exists(out)

    def traps(so):
        sass = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True, check=True).stdout
        return sum(1 for line in sass.splitlines() if "TRAP" in line)

    debug, product = traps(out), traps(gsclib.SO_PATH)
    assert debug >= product + 40, (debug, product)
