"""CPU checks of the C-ABI boundary: the library loads (no GPU needed), every
symbol declared in include/*.h is exported and bound, and the product path
fails loudly without a CUDA device."""

import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*(?:[a-z_]+\s*\**\s+)+(csb_[a-z0-9_]+)\s*\(", txt, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_header_declares_entry_points():
    syms = header_symbols()
    for name in ("csb_residual", "csb_assemble", "csb_lusgs", "csb_implicit_step", "csb_iteration",
                 "csb_status", "csb_set_grid", "csb_set_model"):
        assert name in syms


def test_library_loads_and_exports_every_header_symbol():
    from paper_2403_03440_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2403_03440_b200 import build
        build.build()
    lib = _lib.load()
    assert lib.csb_version() == 1
    for name in header_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == header_symbols()


def test_library_is_sm100a():
    import shutil
    import subprocess
    from paper_2403_03440_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2403_03440_b200 import ExtensionMissing, compute_metrics, generate_box
    from paper_2403_03440_b200.boundary import BoundaryCondition
    from paper_2403_03440_b200.mixture import cloned_mixture, make_primitive, prim_to_cons
    from paper_2403_03440_b200.spatial import assemble_residual
    model = cloned_mixture(2)
    grid = compute_metrics(generate_box(1.0, (2, 2, 1)))
    inf = make_primitive(model, rho=1.0, T=300.0, Y=[0.5, 0.5])
    q = np.broadcast_to(prim_to_cons(inf, model), grid.dims + (model.nvar,)).copy()
    bcs = {f: BoundaryCondition("farfield", freestream=inf)
           for f in ("imin", "imax", "jmin", "jmax", "kmin", "kmax")}
    with pytest.raises(ExtensionMissing):
        assemble_residual(q, grid, bcs, None, model)


def test_product_does_not_import_oracle():
    for path in glob.glob(os.path.join(ROOT, "paper_2403_03440_b200", "*.py")):
        src = open(path).read()
        assert "import oracle" not in src and "from oracle" not in src, path
