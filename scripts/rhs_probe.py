"""Timing probe of the residual kernel: python scripts/rhs_probe.py [ni nj] [ns]"""
import ctypes
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.configs import build_case  # noqa: E402
from paper_2403_03440_b200.device import get_engine  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    ni, nj = (a[0], a[1]) if len(a) >= 2 else (512, 512)
    ns = a[2] if len(a) >= 3 else 5
    spec = C.config0(seed=1, dims=(ni, nj, 1)) if ns == 5 else C.config3(ns, dims=(ni, nj, 1))
    grid, model, bcs, mech = build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    q = eng.to_soa(spec.q, eng.nv)
    R = eng.empty(eng.nv, eng.N)
    st = torch.cuda.current_stream()
    reps = int(os.environ.get("REPS", 10))
    for _ in range(2):
        eng.lib.csb_residual(eng.ctx, q.data_ptr(), R.data_ptr(), None, 0, ctypes.c_void_p(eng.stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        eng.lib.csb_residual(eng.ctx, q.data_ptr(), R.data_ptr(), None, 0, ctypes.c_void_p(eng.stream))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"residual {ni}x{nj} ns={ns}: {ms * 1e3:.1f} us  ({ni * nj / ms * 1e3:.3e} cells/s)", flush=True)


if __name__ == "__main__":
    main()
