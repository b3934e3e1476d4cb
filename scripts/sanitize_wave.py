"""Small driver for compute-sanitizer runs of the 2-D wavefront path: one
implicit iteration (residual, records, forward + backward sweeps, closure)
per scheme (CS1, CS2, CI) on a 48 x 832 box (26 strips of 32 rows), in both
launch orders of csb_wave.cuh (records -> forward sweep serial, and the
overlapped order forced with CSB_FORCE_OVERLAP), plus an 11-species O-grid
with a wall and a 25-strip box with chemistry (CS: per-species diagonal
records; CI: generic hyperplane sweeps + block inverse).  Exits 0 when every call returns CSB_OK.

    compute-sanitizer --tool memcheck python scripts/sanitize_wave.py
"""
import ctypes
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.device import SCHEMES, get_engine  # noqa: E402


def run(spec, schemes):
    grid, model, bcs, mech = C.build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    if eng.chem_on():
        eng.ensure_workspace(True)  # CI with chemistry: species block inverse
    q = eng.to_soa(spec.q, eng.nv).clone()
    qn, R, norms = eng.empty(eng.nv, eng.N), eng.empty(eng.nv, eng.N), eng.empty(4)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for order in ("serial", "forced"):
        os.environ.pop("CSB_FORCE_OVERLAP", None)
        os.environ.pop("CSB_NO_OVERLAP", None)
        os.environ["CSB_FORCE_OVERLAP" if order == "forced" else "CSB_NO_OVERLAP"] = "1"
        for sch in schemes:
            rc = eng.lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), SCHEMES[sch], 0, 0,
                                       qn.data_ptr(), R.data_ptr(), norms.data_ptr(), st)
            assert rc == 0, eng.lib.csb_last_error(eng.ctx)
            torch.cuda.synchronize()
            eng.status()
            print(f"{spec.name} {spec.dims} {sch} {order}: ok", flush=True)


def main():
    run(C.config0(seed=5, dims=(48, 832, 1)), ("CS1", "CS2", "CI"))
    run(C.config2(seed=6, dims=(40, 96, 1), sigma=1.5), ("CS1", "CI"))
    run(C.config3(5, seed=7, dims=(24, 800, 1), chemistry=True), ("CS1", "CI"))


if __name__ == "__main__":
    main()
