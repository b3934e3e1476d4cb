"""Debug: device march vs host loop on the reference cylinder case."""
import os, sys
ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from test_gpu_march import binary_model, cylinder_case
from paper_2403_03440_b200.driver import steady_solve

for orders in (np.inf, 1.0, 3.0):
    case = cylinder_case(binary_model(), "CS1", max_iters=120, residual_drop_orders=orders)
    qd, hd = steady_solve(case)
    qh, hh = steady_solve(case, device_march=False)
    print("orders", orders, "device", hd.reason, len(hd.iters), "host", hh.reason, len(hh.iters))
    n = min(len(hd.iters), len(hh.iters))
    rd, rh = np.array(hd.res_density[:n]), np.array(hh.res_density[:n])
    print(" max rel dens diff", np.max(np.abs(rd - rh) / rh), "cfl eq", hd.cfl[:n] == hh.cfl[:n],
          "retries", sum(hd.retries), sum(hh.retries))
    print(" dens first/last", rd[0], rd[-1], rh[0], rh[-1])
    print(" dev head", rd[:5], "host head", rh[:5])
