"""Config 4 (BASELINE.json): steady pseudo-time march on a curvilinear O-grid
with 11 species, freestream start, CFL ramp 1 -> 1000 (x2 every 45
iterations), through the drop-in steady_solve.  Reports sustained accepted
cell-iterations/s (retried implicit steps cost time but do not
count), retries, and the residual history.

    python scripts/march_config4.py [ni nj iters]      (default 4096 2048 500)
"""
import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200.configs import build_case  # noqa: E402
from paper_2403_03440_b200.driver import Case, steady_solve  # noqa: E402
from paper_2403_03440_b200.mixture import make_primitive  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    ni, nj, iters = (a + [4096, 2048, 500][len(a):])[:3]
    t0 = time.perf_counter()
    spec = C.config4(dims=(ni, nj, 1))
    grid, model, bcs, mech = build_case(spec)
    rho, u, T, Y = spec.bcs["jmax"].fs
    inf = make_primitive(model, rho=rho, u=u, T=T, Y=Y)
    r0, r1, r2 = spec.extra["cfl_ramp"]
    case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, mech=mech, scheme="CS1",
                cfl=spec.cfl, cfl_ramp=(r0, r1, int(r2)), max_iters=iters,
                residual_drop_orders=np.inf, stop_on_absolute_floor=False)
    setup = time.perf_counter() - t0
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    q, hist = steady_solve(case, spec.q, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t1
    N = ni * nj
    accepted = len(hist.iters)
    out = {"config": "config4", "grid": f"{ni}x{nj}", "ns": 11, "iterations": accepted,
           "retries": int(sum(hist.retries)), "wall_s": wall, "setup_s": setup,
           "sustained_cell_it_per_s": N * accepted / wall,
           "implicit_s": float(sum(hist.implicit_seconds)),
           "cfl_final": hist.cfl[-1] if hist.cfl else None,
           "res_density_first_last": [hist.res_density[0], hist.res_density[-1]],
           "res_flow_every_50": hist.res_flow[::50], "reason": hist.reason}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
