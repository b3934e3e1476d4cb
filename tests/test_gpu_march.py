"""The device-resident steady march (csb_march_*: one CUDA graph per chunk,
every loop decision on the device) against the host-driven loop and the
reference driver's own known-answer tests (pkg/tests/test_driver.py:24-50,
108-147).  The golden-history tests in test_gpu_parity.py (CS1 and CI
cylinder marches, reduced config 4) also run through the device march, the
default of steady_solve.
"""

import numpy as np
import pytest

from golden_cases import get
from product_cases import golden_product

pytestmark = pytest.mark.gpu


def _P():
    import paper_2403_03440_b200 as P
    return P


def binary_model():
    P = _P()
    return P.MixtureModel([P.SpeciesData("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0),
                           P.SpeciesData("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)])


def cylinder_case(model, scheme, dims=(16, 12, 1), cfl=5.0, mach=2.0, **kw):
    """pkg/tests/test_driver.py:108-123."""
    P = _P()
    from paper_2403_03440_b200.boundary import BoundaryCondition
    from paper_2403_03440_b200.driver import Case
    grid = P.compute_metrics(P.generate_cylinder_ogrid(0.045, 0.25, dims, stretch=1.15))
    Y = np.full(model.ns, 1.0 / model.ns)
    chill = P.make_primitive(model, rho=1.0, T=250.0, Y=Y)
    inf = P.make_primitive(model, rho=1.0, T=250.0, u=(mach * float(chill.c), 0.0, 0.0), Y=Y)
    bcs = {"imin": BoundaryCondition("supersonic_outflow"),
           "imax": BoundaryCondition("supersonic_outflow"),
           "jmin": BoundaryCondition("noslip_isothermal", T_wall=300.0),
           "jmax": BoundaryCondition("farfield", freestream=inf),
           "kmin": BoundaryCondition("symmetry"), "kmax": BoundaryCondition("symmetry")}
    return Case(grid=grid, model=model, bcs=bcs, freestream=inf, scheme=scheme, cfl=cfl, **kw)


def box_case(model, dims=(6, 5, 4), scheme="CI", **kw):
    """pkg/tests/test_driver.py:24-29."""
    P = _P()
    from paper_2403_03440_b200.boundary import BoundaryCondition
    from paper_2403_03440_b200.driver import Case
    grid = P.compute_metrics(P.generate_box(1.0, dims))
    Y = np.full(model.ns, 1.0 / model.ns)
    inf = P.make_primitive(model, rho=1.0, u=(180.0, -40.0, 20.0), T=300.0, Y=Y)
    bcs = {f: BoundaryCondition("farfield", freestream=inf)
           for f in ("imin", "imax", "jmin", "jmax", "kmin", "kmax")}
    return Case(grid=grid, model=model, bcs=bcs, freestream=inf, scheme=scheme, **kw)


def _same_history(a, b):
    """Same iterations, stop, CFL trajectory and retries; the norms agree to
    the last bits (the device march reduces them inside the residual kernel,
    the host loop in a separate reduction: different summation order)."""
    assert a.iters == b.iters
    assert a.reason == b.reason
    for key in ("cfl", "retries"):
        assert np.array_equal(np.asarray(getattr(a, key)), np.asarray(getattr(b, key))), key
    for key in ("res_flow", "res_species", "res_density"):
        np.testing.assert_allclose(getattr(a, key), getattr(b, key), rtol=1e-13, atol=0, err_msg=key)
    qa, qb = np.asarray(a.q_stag, float), np.asarray(b.q_stag, float)
    assert np.array_equal(qa, qb, equal_nan=True)


def test_device_march_equals_host_loop_with_retries():
    """Reduced config 4 (11 species, freestream start, CFL ramp x2 every 8
    iterations, 40 iterations): CFL halvings, recoveries, the wall monitor
    and the residual histories of the device march equal the host loop's
    bit for bit."""
    from paper_2403_03440_b200.driver import Case, steady_solve
    name = "march_c4"
    grid, model, bcs, mech, q0, cfl = golden_product(name)
    f = get(name, "fs_prim")
    inf = _P().make_primitive(model, rho=f[0], u=f[1:4], T=f[4], Y=f[5:])
    case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, mech=mech, scheme="CS1",
                cfl=1000.0, cfl_ramp=(1.0, 2.0, 8), max_iters=40, residual_drop_orders=np.inf,
                stop_on_absolute_floor=False)
    qd, hd = steady_solve(case, q0)
    qh, hh = steady_solve(case, q0, device_march=False)
    assert sum(hd.retries) > 0  # the case exercises the device retry loop
    _same_history(hd, hh)
    assert np.array_equal(qd, qh)


@pytest.mark.parametrize("scheme", ["CI", "CS1", "CS2"])
def test_cylinder_mini_convergence(scheme):
    """pkg/tests/test_driver.py:126-133 with a 1-order drop: the reference
    itself reaches only ~2.5 orders in 600 iterations for CS1 (its test
    expects 3 and is one of the suite's failing tests), so the
    stop is exercised at 1 order and checked against the host loop."""
    from paper_2403_03440_b200.driver import steady_solve
    case = cylinder_case(binary_model(), scheme, max_iters=600, residual_drop_orders=1.0)
    q, hist = steady_solve(case)
    assert hist.reason == "converged_residual_drop"
    assert hist.res_density[-1] <= hist.res_density[0] * 1e-1
    qh, hh = steady_solve(case, device_march=False)
    _same_history(hist, hh)
    assert np.array_equal(q, qh)


def test_cfl_ramp_schedule_recorded():
    """pkg/tests/test_driver.py:136-147."""
    from paper_2403_03440_b200.driver import steady_solve
    base = dict(max_iters=400, residual_drop_orders=1.0)  # (3 in the reference's failing test)
    _, hist_fixed = steady_solve(cylinder_case(binary_model(), "CI", cfl=5.0, **base))
    ramped = cylinder_case(binary_model(), "CI", cfl=20.0, **base)
    ramped.cfl_ramp = (5.0, 2.0, 50)
    _, hist_ramp = steady_solve(ramped)
    for it, c in zip(hist_ramp.iters, hist_ramp.cfl):
        assert c == pytest.approx(min(20.0, 5.0 * 2.0 ** ((it - 1) // 50)))
    assert hist_ramp.reason == "converged_residual_drop"
    assert hist_ramp.iters[-1] <= hist_fixed.iters[-1]


def test_uniform_freestream_terminates_immediately():
    """pkg/tests/test_driver.py:32-37: the absolute floor stops iteration 1."""
    from paper_2403_03440_b200.driver import steady_solve
    case = box_case(binary_model())
    q, hist = steady_solve(case)
    assert len(hist.iters) == 1
    assert hist.reason == "converged_absolute"
    np.testing.assert_array_equal(q, case.initial_field())


@pytest.mark.parametrize("scheme", ["CI", "CS1", "CS2"])
def test_uniform_freestream_fixed_point_device_march(scheme):
    """pkg/tests/test_driver.py:40-50 through the device march (3-D box:
    generic hyperplane sweeps inside the graph)."""
    from paper_2403_03440_b200.driver import steady_solve
    case = box_case(binary_model(), dims=(5, 4, 3), scheme=scheme, max_iters=50,
                    residual_drop_orders=np.inf, stop_on_absolute_floor=False)
    q0 = case.initial_field()
    q, hist = steady_solve(case)
    assert hist.reason == "max_iters" and len(hist.iters) == 50
    assert np.max(np.abs(q - q0)) <= 1e-11 * np.max(np.abs(q0))


def test_monitor_plateau_stop_matches_host_loop():
    """The heat-flux monitor plateau stop (driver.py:300-306): sampled by the
    host between device chunks, decided at the same iteration as the host
    loop."""
    from paper_2403_03440_b200.driver import steady_solve
    case = cylinder_case(binary_model(), "CS1", max_iters=300, residual_drop_orders=np.inf,
                         monitor_every=5, monitor_window=4, monitor_rel_change=0.5)
    qd, hd = steady_solve(case)
    qh, hh = steady_solve(case, device_march=False)
    assert hd.reason == "converged_monitor_plateau"
    _same_history(hd, hh)
    assert np.array_equal(qd, qh)


def test_diverged_after_retries_like_reference():
    """config 2's smoothed random field at CFL 100 fails
    admissibility next to the 300 K wall at every halving; the reference
    raises Diverged on the first step.  The device march does too."""
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.driver import Case, steady_solve
    from paper_2403_03440_b200.errors import Diverged
    spec = C.config2(seed=12, dims=(24, 20, 1), sigma=1.5)
    grid, model, bcs, mech = C.build_case(spec)
    case = Case(grid=grid, model=model, bcs=bcs, freestream=C.freestream_of(spec, model),
                scheme="CS1", cfl=100.0, max_iters=10, residual_drop_orders=np.inf,
                stop_on_absolute_floor=False)
    with pytest.raises(Diverged):
        steady_solve(case, spec.q)
    with pytest.raises(Diverged):
        steady_solve(case, spec.q, device_march=False)
