"""Profiling driver: a few fused implicit iterations (csb_iteration) on one
config, for ncu captures of the per-iteration kernels.

    python scripts/prof_iter.py [config] [ns] [iters] [scheme]
      config 1: 512^2 air5 box; config 3: 1024^2 box with ns species;
      config 2: 1024^2 O-grid ns=11; config 4: 4096x2048 O-grid ns=11
      (freestream start state at the ramp's first CFL)
      scheme CS1 (default) | CI

Run it once plainly (exit 0), then under
    ncu --set full --import-source on -k regex:"k_residual|k_records2d|k_wave2d|k_epilogue2d" -s 5 -c 5
(-s 5 skips the first iteration's kernels: cold model tables).
"""

import ctypes
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.device import SCHEMES, get_engine  # noqa: E402


def main():
    if os.environ.get("CSB_L2_FETCH"):  # experiment: cudaLimitMaxL2FetchGranularity (0x05)
        torch.cuda.init()
        torch.zeros(1, device="cuda")
        rt = ctypes.CDLL("libcudart.so")
        rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(int(os.environ["CSB_L2_FETCH"])))
        v = ctypes.c_size_t(0)
        rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        print("L2 fetch granularity", rc, v.value)
    a = sys.argv[1:]
    cfg = int(a[0]) if a else 1
    ns = int(a[1]) if len(a) > 1 else 11
    iters = int(a[2]) if len(a) > 2 else 3
    scheme = a[3] if len(a) > 3 else "CS1"
    if cfg == 4:
        spec = C.config4()
        spec.cfl = 1.0
    elif cfg == 2:
        spec = C.config2()
    else:
        spec = C.config1(seed=1) if cfg == 1 else C.config3(ns, seed=3)
    grid, model, bcs, mech = C.build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    q = eng.to_soa(spec.q, eng.nv).clone()
    qn = eng.empty(eng.nv, eng.N)
    R = eng.empty(eng.nv, eng.N)
    norms = eng.empty(4)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
    ev[0].record()
    for k in range(iters):
        rc = eng.lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), SCHEMES[scheme], 0, 0,
                                   qn.data_ptr(), R.data_ptr(), norms.data_ptr(), st)
        assert rc == 0, eng.lib.csb_last_error(eng.ctx)
        ev[k + 1].record()
    torch.cuda.synchronize()
    eng.status()
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(iters)]
    print(f"config{cfg} ns={spec.ns} {spec.dims} {scheme}: ms/iteration {ms}")


if __name__ == "__main__":
    main()
