"""Run one 2-D wavefront implicit step on a few small grids (sanitizer target)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2403_03440_b200 import configs as C  # noqa: E402
from paper_2403_03440_b200 import driver, spatial  # noqa: E402
from paper_2403_03440_b200.configs import build_case  # noqa: E402

for dims in [(8, 6, 1), (40, 45, 1), (3, 70, 1)]:
    spec = C.config0(seed=7, dims=dims)
    grid, model, bcs, mech = build_case(spec)
    R = spatial.assemble_residual(spec.q, grid, bcs, mech, model)
    case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, scheme="CS1", cfl=spec.cfl)
    qn, flags, cnt, cell = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=2)
    print(dims, "flags", flags, "gate failures", cnt, flush=True)
