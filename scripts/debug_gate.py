import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import oracle as O
from golden_cases import get, thermo
from product_cases import golden_product
from paper_2403_03440_b200 import driver
for case, key in [("box_air5", "CI"), ("box_air5", "CS1"), ("thin", "CS2")]:
    grid, model, bcs, mech, q, cfl = golden_product(case)
    c = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=key, cfl=cfl)
    qn, flags, cnt, cell = driver.implicit_step_raw(c, q, get(case, "R"), cfl)
    th = thermo(case)
    bad_dev_o = O.update(q, qn - q, key, th)[1]  # oracle gate on device q_new (approx)
    gold = get(case, key + "/gate_bad")
    qg = get(case, key + "/q_new")
    pr_dev = O.decode(qn, th, raise_on_bad=False)
    pr_gold = O.decode(qg, th, raise_on_bad=False)
    print(case, key, "flags", flags, "cnt", cnt, "gold", gold.sum(), "oracle-on-dev", bad_dev_o.sum(),
          "decode-bad dev", pr_dev.bad.sum(), "decode-bad gold", pr_gold.bad.sum())
    print("  max|qn-qg|/max|qg| per comp", np.max(np.abs(qn - qg), axis=(0,1,2)) / np.max(np.abs(qg), axis=(0,1,2)))
