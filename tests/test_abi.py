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
    """Every product entry point needs the sm_100a library on a CUDA device:
    without one it raises ExtensionMissing instead of computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import oracle as O
    from paper_2403_03440_b200 import (ExtensionMissing, compute_metrics, configs, generate_box,
                                       generate_cylinder_ogrid, make_primitive)
    from paper_2403_03440_b200.boundary import BoundaryCondition
    from paper_2403_03440_b200.driver import wall_heat_flux
    from paper_2403_03440_b200.spatial import assemble_residual
    model = configs.cloned_mixture(2)
    nodes = configs.box_nodes(1.0, (2, 2, 1))
    host_grid = O.Grid(nodes)  # reference-shaped attributes (duck typing)
    q = np.ones(host_grid.dims + (model.nvar,))
    calls = [lambda: generate_box(1.0, (2, 2, 1)),
             lambda: generate_cylinder_ogrid(1.0, 2.0, (4, 4, 1)),
             lambda: compute_metrics(nodes),
             lambda: make_primitive(model, rho=1.0, T=300.0, Y=[0.5, 0.5])]
    for call in calls:
        with pytest.raises(ExtensionMissing):
            call()
    bcs = {f: BoundaryCondition("supersonic_outflow")
           for f in ("imin", "imax", "jmin", "jmax", "kmin", "kmax")}
    with pytest.raises(ExtensionMissing):
        assemble_residual(q, host_grid, bcs, None, model)
    bcs["jmin"] = BoundaryCondition("noslip_isothermal", T_wall=300.0)
    with pytest.raises(ExtensionMissing):
        wall_heat_flux(q, host_grid, bcs, model)


def test_plot3d_is_host_io():
    """Plot3D I/O is file parsing (no device): round trip and error offsets
    (reference pkg/tests/test_grid.py:100-143)."""
    import numpy as np
    from paper_2403_03440_b200 import MultiBlockUnsupported, ParseError, configs
    from paper_2403_03440_b200.plot3d import read_plot3d, write_plot3d
    import tempfile
    d = tempfile.mkdtemp()
    nodes = configs.box_nodes((1.0, 2.0, 0.5), (4, 3, 2))
    nodes += 1e-3 * np.sin(nodes * 7.0)
    path = os.path.join(d, "g.xyz")
    write_plot3d(path, nodes)
    np.testing.assert_array_equal(read_plot3d(path), nodes)
    lines = open(path).read().splitlines()
    open(path, "w").write("\n".join(lines[1:]) + "\n")  # headerless single block
    np.testing.assert_array_equal(read_plot3d(path), nodes)
    write_plot3d(path, configs.box_nodes(1.0, (3, 3, 3)))
    text = open(path).read()
    open(path, "w").write(text[: len(text) // 2])
    with pytest.raises(ParseError):
        read_plot3d(path)
    open(path, "w").write("2\n2 2 2\n2 2 2\n" + "0.0\n" * 48)
    with pytest.raises(MultiBlockUnsupported):
        read_plot3d(path)
    open(path, "w").write("1\n2 2 oops\n")
    with pytest.raises(ParseError) as err:
        read_plot3d(path)
    assert err.value.byte_offset == 6
    open(path, "w").write("1\n# dims next\n1 1 1 # one node\n0.5 # x\n1.5\n2.5\n")
    np.testing.assert_array_equal(read_plot3d(path), [[[[0.5, 1.5, 2.5]]]])
    open(path, "w").write("1\n1 1 1\n0.5 1.5 2.5 3.5\n")
    with pytest.raises(ParseError) as err:
        read_plot3d(path)
    assert err.value.byte_offset == len("1\n1 1 1\n0.5 1.5 2.5 ")


def test_product_does_not_import_oracle():
    for path in glob.glob(os.path.join(ROOT, "paper_2403_03440_b200", "*.py")):
        src = open(path).read()
        assert "import oracle" not in src and "from oracle" not in src, path
