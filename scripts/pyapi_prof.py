"""Timing breakdown of the numpy drop-in calls at config 4 (assemble_residual,
_implicit_step) and of the host <-> device copies under them.

    python scripts/pyapi_prof.py
"""
import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2403_03440_b200 import configs as C, spatial, driver
from paper_2403_03440_b200.device import get_engine
spec = C.config4(); spec.cfl = 1.0
grid, model, bcs, mech = C.build_case(spec)
q = np.ascontiguousarray(spec.q)
case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme="CS1", cfl=spec.cfl)
eng = get_engine(grid, model)
def T(f, n=4):
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(n): r=f()
    torch.cuda.synchronize(); return (time.perf_counter()-t)/n, r
R = spatial.assemble_residual(q, grid, bcs, mech, model)
t, _ = T(lambda: spatial.assemble_residual(q, grid, bcs, mech, model)); print("assemble_residual", t)
t, _ = T(lambda: driver._implicit_step(case, q, R, spec.cfl)); print("_implicit_step", t)
t, qs = T(lambda: eng.to_soa(q, eng.nv)); print("to_soa", t)
t, x = T(lambda: torch.from_numpy(q)); print("from_numpy", t)
t, xd = T(lambda: x.to("cuda")); print("pageable H2D", t)
t, _ = T(lambda: eng.from_soa(qs, q, q.shape)); print("from_soa", t)
t, h = T(lambda: xd.cpu()); print("pageable D2H", t)
t, _ = T(lambda: h.numpy()); print("numpy()", t)
pin = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
t, _ = T(lambda: pin.copy_(x)); print("host memcpy to pinned", t)
t, _ = T(lambda: xd.copy_(pin, non_blocking=True)); print("pinned H2D", t)
t, _ = T(lambda: pin.copy_(xd, non_blocking=True)); print("pinned D2H", t)
torch.set_num_threads(8)
t, _ = T(lambda: pin.copy_(x)); print("host memcpy to pinned (8 threads)", t)
t, _ = T(lambda: np.copyto(h.numpy(), pin.numpy())); print("np.copyto pinned->pageable", t)
