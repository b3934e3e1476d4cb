"""Per-stage CUDA-event times of one implicit iteration for a few configs,
for A/B comparison of library builds (load a variant with CSB_LIB_PATH).

    CSB_LIB_PATH=_variants/<tag>/libcsflow_b200.so python scripts/stage_times.py [cfg ...]
      cfg: c4 (4096x2048 O-grid ns=11), c3_<ns> (1024^2 box), c1 (512^2 air5)
      CSB_SCHEME=0|1|2 picks CI / CS1 (default) / CS2
"""
import ctypes
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.device import get_engine  # noqa: E402


def spec_of(name):
    if name == "c4":
        s = C.config4()
        s.cfl = 1.0
        return s
    if name == "c1":
        return C.config1(seed=1)
    if name.startswith("c3_"):
        return C.config3(int(name[3:]), seed=3)
    if name == "c2":
        return C.config2()
    raise SystemExit(name)


def main():
    if os.environ.get("CSB_L2_FETCH"):  # experiment: cudaLimitMaxL2FetchGranularity (0x05)
        torch.cuda.init()
        torch.zeros(1, device="cuda")
        rt = ctypes.CDLL("libcudart.so")
        rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(int(os.environ["CSB_L2_FETCH"])))
        v = ctypes.c_size_t(0)
        rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
        print("L2 fetch granularity", rc, v.value)
    names = sys.argv[1:] or ["c4"]
    out = {"lib": os.environ.get("CSB_LIB_PATH", "default")}
    for name in names:
        spec = spec_of(name)
        grid, model, bcs, mech = C.build_case(spec)
        eng = get_engine(grid, model)
        eng.set_bcs(bcs)
        eng.set_mechanism(mech)
        q = eng.to_soa(spec.q, eng.nv).clone()
        qn, R, norms = eng.empty(eng.nv, eng.N), eng.empty(eng.nv, eng.N), eng.empty(4)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        lib = eng.lib
        sch = int(os.environ.get("CSB_SCHEME", "1"))  # 1 CS1, 2 CS2, 0 CI
        for _ in range(3):
            assert lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), sch, 0, 0, qn.data_ptr(),
                                     R.data_ptr(), norms.data_ptr(), st) == 0
        torch.cuda.synchronize()
        K = 5
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        for _ in range(K):
            lib.csb_residual(eng.ctx, q.data_ptr(), R.data_ptr(), None, 0, st)
        b.record()
        for _ in range(K):
            lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), sch, 0, 0, qn.data_ptr(),
                              R.data_ptr(), norms.data_ptr(), st)
        c.record()
        torch.cuda.synchronize()
        ms5 = (ctypes.c_float * 5)()
        for _ in range(2):
            lib.csb_profile_step(eng.ctx, q.data_ptr(), R.data_ptr(), float(spec.cfl), sch,
                                 qn.data_ptr(), ms5, st)
        eng.status()
        out[name] = {"residual_ms": a.elapsed_time(b) / K, "iteration_ms": b.elapsed_time(c) / K,
                     "records_ms": ms5[1], "fwd_ms": ms5[2], "bwd_ms": ms5[3], "epilogue_ms": ms5[4]}
        del eng, q, qn, R
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
