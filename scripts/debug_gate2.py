import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from golden_cases import get, has
from product_cases import golden_product
from paper_2403_03440_b200 import driver, implicit, lusgs
for case, key in [("box_air5", "CS2"), ("thin", "CS2"), ("ogrid_air11", "CS1")]:
    grid, model, bcs, mech, q, cfl = golden_product(case)
    c = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=key, cfl=cfl)
    qn, flags, cnt, cell = driver.implicit_step_raw(c, q, get(case, "R"), cfl)
    print(case, key, "fresh: cnt", cnt, "gold", int(get(case, key + "/gate_bad").sum()), "flags", flags)
    op = implicit.assemble_lhs(q, grid, key, get(case, "dtau"), mech, model)
    dq, star = lusgs.lusgs_solve(op, -get(case, "R"), return_forward=True)
    qn2, flags2, cnt2, cell2 = driver.implicit_step_raw(c, q, get(case, "R"), cfl)
    print("   after assemble+lusgs: cnt", cnt2, "flags", flags2, "maxdiff", np.nanmax(np.abs(qn2 - qn)))
    qn3, flags3, cnt3, cell3 = driver.implicit_step_raw(c, q, get(case, "R"), cfl)
    print("   again: cnt", cnt3, "flags", flags3)
