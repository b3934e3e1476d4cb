"""Timing probe of the 2-D wavefront implicit step over grid shapes.

    python scripts/wave_probe.py [ni nj ...]

Prints per-stage device ms (csb_profile_step) and the per-step cost of the
sweep (ms / (T + strip pipeline)), to separate per-step latency from the
strip hand-off cost.
"""

import ctypes
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.configs import build_case  # noqa: E402
from paper_2403_03440_b200.device import get_engine  # noqa: E402
from paper_2403_03440_b200.spatial import residual_device  # noqa: E402


def probe(ni, nj, ns=5, reps=int(os.environ.get("REPS", 5))):
    spec = C.config0(seed=1, dims=(ni, nj, 1)) if ns == 5 else C.config3(ns, dims=(ni, nj, 1))
    grid, model, bcs, mech = build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    q = eng.to_soa(spec.q, eng.nv)
    R, _ = residual_device(eng, q)
    qn = eng.empty(eng.nv, eng.N)
    ms5 = (ctypes.c_float * 5)()
    acc = [0.0] * 5
    for r in range(reps + 1):
        rc = eng.lib.csb_profile_step(eng.ctx, q.data_ptr(), R.data_ptr(), float(spec.cfl), 1,
                                      qn.data_ptr(), ms5, ctypes.c_void_p(eng.stream))
        assert rc == 0, eng.lib.csb_last_error(eng.ctx)
        if r:
            for k in range(5):
                acc[k] += ms5[k] / reps
    eng.status()
    nstrip = (nj + 31) // 32
    T = ((ni + 31 + 15) // 16) * 16
    fwd = acc[2]
    print(f"{ni:5d}x{nj:<5d} ns={ns:2d} strips={nstrip:3d} T={T:5d}  records {acc[1]*1e3:8.1f} us  "
          f"fwd {fwd*1e3:8.1f} us  bwd {acc[3]*1e3:8.1f} us  epi {acc[4]*1e3:7.1f} us  "
          f"fwd/T {fwd*1e6/T:7.1f} ns/step", flush=True)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    shapes = list(zip(args[0::2], args[1::2])) if args else [
        (512, 32), (2048, 32), (512, 64), (512, 128), (512, 256), (512, 512), (1024, 1024)]
    for ni, nj in shapes:
        probe(ni, nj, ns=int(os.environ.get("NS", 5)))
    if not args:
        probe(512, 512, ns=11)
