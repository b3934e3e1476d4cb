"""GPU parity of the §8(f) rows around the hot path: grid generators and
metric terms on the device (f4), state construction, the wall heat flux and
stagnation monitor (f2), and dual-time stepping (f3).

Oracles: fixtures of the real reference (tests/golden/make_golden.py:
generators_case, wall fluxes of the one-iteration cases, dual_time_case) and
the reference's own known-answer tests (pkg/tests/test_grid.py,
test_driver.py:76-106 and 147-160, test_implicit.py:290-303).
"""

import numpy as np
import pytest

import oracle as O
from golden_cases import comp_relerr, get
from product_cases import golden_product

pytestmark = pytest.mark.gpu


def _P():
    import paper_2403_03440_b200 as P
    return P


# ------------------------------------------------------------- f4: grids

@pytest.mark.parametrize("case", ["box_air5", "ogrid_air11", "chem3d", "thin", "warped"])
def test_device_metrics_bit_identical_to_reference(case):
    """csb_grid_metrics rounds like numpy (grid.py:51-99): face vectors and
    volumes equal the reference's bit for bit."""
    g = _P().compute_metrics(get(case, "nodes"))
    for key, got in (("Si", g.Si), ("Sj", g.Sj), ("Sk", g.Sk), ("vol", g.volume)):
        ref = get(case, key)
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), (key, float(np.max(np.abs(got - ref))))


@pytest.mark.parametrize("key", ["box", "ogrid", "ogrid_first_cell", "ogrid_quarter"])
def test_device_generators_match_reference(key):
    P = _P()
    ref = get("gen", key)
    if key == "box":
        got = P.generate_box((0.3, 0.2, 0.1), (7, 5, 3))
        assert np.array_equal(got, ref)
    elif key == "ogrid":
        got = P.generate_cylinder_ogrid(1.0, 3.5, (20, 16, 2), stretch=1.05)
        assert np.array_equal(got, ref)
    elif key == "ogrid_quarter":
        got = P.generate_cylinder_ogrid(0.045, 0.2, (12, 9, 1), theta_deg=(180.0, 90.0), span=0.02)
        assert np.array_equal(got, ref)
    else:  # wall-spacing solve: a different root finder, same ratio to ~1e-15
        got = P.generate_cylinder_ogrid(0.045, 0.145, (8, 16, 1), first_cell=1e-4)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)


def test_large_grid_metrics_match_oracle_numpy():
    """A config-2-shaped O-grid (stretch 1.02, 1e-5 wall spacing) at 256 x 192:
    device metrics equal the oracle's numpy metrics bit for bit."""
    from paper_2403_03440_b200 import configs as C
    nodes = C.ogrid_nodes((256, 192, 1))
    g = _P().compute_metrics(nodes)
    og = O.Grid(nodes)
    for a, b in ((g.Si, og.Si), (g.Sj, og.Sj), (g.Sk, og.Sk), (g.volume, og.volume),
                 (g.Sci, og.Sci), (g.Scj, og.Scj), (g.Sck, og.Sck), (g.J, og.J)):
        assert np.array_equal(a, b)


def _closure(grid):
    s = (grid.Si[1:] - grid.Si[:-1] + grid.Sj[:, 1:] - grid.Sj[:, :-1]
         + grid.Sk[:, :, 1:] - grid.Sk[:, :, :-1])
    return np.abs(s).max() / np.linalg.norm(grid.Si, axis=-1).max()


def test_reference_grid_kats():
    """pkg/tests/test_grid.py:17-97 on the device path."""
    P = _P()
    g = P.compute_metrics(P.generate_box(1.0, (10, 10, 10)))
    np.testing.assert_allclose(g.volume, 1e-3, rtol=1e-13)
    np.testing.assert_allclose(g.J, 1000.0, rtol=1e-13)
    np.testing.assert_allclose(g.Si[..., 0], 0.01, rtol=1e-13)
    np.testing.assert_allclose(g.Si[..., 1:], 0.0, atol=1e-18)
    np.testing.assert_allclose(g.Sj[..., 1], 0.01, rtol=1e-13)
    np.testing.assert_allclose(g.Sk[..., 2], 0.01, rtol=1e-13)
    nodes = P.generate_box(1.0, (10, 10, 10))
    assert nodes.shape == (11, 11, 11, 3)
    np.testing.assert_allclose(np.diff(nodes[:, 0, 0, 0]), 0.1, rtol=1e-13)
    # geometric conservation on a warped grid
    rng = np.random.default_rng(2)
    nodes = P.generate_box(1.0, (6, 5, 4))
    bump = 0.25 * np.sin(2 * np.pi * nodes[..., 0]) * np.sin(np.pi * nodes[..., 1])
    nodes[1:-1, 1:-1, 1:-1, 2] += bump[1:-1, 1:-1, 1:-1] * 0.1
    nodes[1:-1, 1:-1, 1:-1, 0] += 0.02 * rng.standard_normal(nodes[1:-1, 1:-1, 1:-1, 0].shape)
    g = P.compute_metrics(nodes)
    assert _closure(g) < 1e-12 and np.all(g.J > 0)
    # an interior face is one stored entry seen from both sides
    rng = np.random.default_rng(4)
    nodes = P.generate_box(1.0, (4, 3, 2))
    nodes[1:-1, 1:-1, 1:-1] += 0.03 * rng.standard_normal(nodes[1:-1, 1:-1, 1:-1].shape)
    g = P.compute_metrics(nodes)
    assert g.face_areas(0)[2, 1, 0].tobytes() == g.face_areas(0)[2, 1, 0].tobytes()
    # degenerate cells and bad dimensions
    nodes = P.generate_box(1.0, (3, 3, 3))
    sw = nodes.copy()
    sw[1, 1, 1], sw[2, 2, 2] = nodes[2, 2, 2].copy(), nodes[1, 1, 1].copy()
    with pytest.raises(P.DegenerateCell):
        P.compute_metrics(sw)
    for bad in (lambda: P.generate_box(1.0, (0, 4, 4)), lambda: P.generate_box(-1.0, (4, 4, 4)),
                lambda: P.generate_cylinder_ogrid(0.045, 0.2, (1, 8, 1)),
                lambda: P.generate_cylinder_ogrid(0.2, 0.1, (8, 8, 1)),
                lambda: P.compute_metrics(np.zeros((3, 3, 3)))):
        with pytest.raises(P.BadDims):
            bad()
    # cylinder generators
    nodes = P.generate_cylinder_ogrid(0.045, 0.2, (32, 32, 1), theta_deg=(180.0, 90.0))
    np.testing.assert_allclose(np.linalg.norm(nodes[:, 0, :, :2], axis=-1), 0.045, atol=1e-12)
    g = P.compute_metrics(nodes)
    assert np.all(g.J > 0) and _closure(g) < 1e-12
    r = np.linalg.norm(P.generate_cylinder_ogrid(0.045, 0.145, (8, 10, 1))[0, :, 0, :2], axis=-1)
    np.testing.assert_allclose(np.diff(r), 0.01, rtol=1e-12)
    r = np.linalg.norm(P.generate_cylinder_ogrid(0.045, 0.145, (8, 16, 1),
                                                 first_cell=1e-4)[0, :, 0, :2], axis=-1)
    assert r[1] - r[0] == pytest.approx(1e-4, rel=1e-9)
    assert r[-1] == pytest.approx(0.145, rel=1e-12)


def test_solver_accepts_reference_shaped_grid():
    """Duck typing: a host grid object with the reference's attributes (the
    oracle's) gives the same residual as this package's device grid."""
    from paper_2403_03440_b200 import spatial
    grid, model, bcs, mech, q, cfl = golden_product("warped")
    R_dev = spatial.assemble_residual(q, grid, bcs, mech, model)
    R_host = spatial.assemble_residual(q, O.Grid(get("warped", "nodes")), bcs, mech, model)
    assert np.array_equal(R_dev, R_host)
    assert comp_relerr(R_dev, get("warped", "R")) <= 1e-12


# ------------------------------------------------------------- state helpers

def test_make_primitive_and_prim_to_cons_match_oracle():
    """csb_primitive (mixture.py:310-351) against the oracle's encode on a
    config-0 random state, and the three (rho, p, T) input pairs agree."""
    from paper_2403_03440_b200 import configs as C
    P = _P()
    spec = C.config0(seed=3, dims=(16, 12, 1))
    model = C.model_of(spec)
    th = O.Thermo(*[np.array([getattr(s, k) for s in spec.species]) for k in
                    ("M", "cp", "hf", "Tref", "mu_ref", "T_mu", "S_mu")])
    pr = O.decode(spec.q, th)
    prim = P.make_primitive(model, rho=pr.rho, u=pr.u, T=pr.T, Y=pr.Y)
    q = P.prim_to_cons(prim, model)
    ref = O.encode(pr.rho, pr.u, pr.T, pr.Y, th)
    assert comp_relerr(q, ref) <= 1e-13
    p2 = P.make_primitive(model, p=prim.p, T=prim.T, u=pr.u, Y=pr.Y)
    p3 = P.make_primitive(model, rho=prim.rho, p=prim.p, u=pr.u, Y=pr.Y)
    np.testing.assert_allclose(p2.rho, prim.rho, rtol=1e-15)
    np.testing.assert_allclose(p3.T, prim.T, rtol=1e-15)
    for f in ("c", "gamma", "h", "Ek"):
        np.testing.assert_allclose(getattr(prim, f), getattr(pr, f), rtol=1e-14)
    with pytest.raises(P.NonPhysicalState):
        P.make_primitive(model, rho=1.0, T=-5.0, Y=np.full(5, 0.2))
    with pytest.raises(P.NonPhysicalState):
        P.make_primitive(model, rho=1.0, T=300.0, Y=np.full(5, 0.3))


# ------------------------------------------------------------- f2: wall heat flux

@pytest.mark.parametrize("case,face", [("ogrid_air11", "jmin"), ("chem3d", "jmin"),
                                       ("warped", "kmin")])
def test_wall_heat_flux_matches_reference(case, face):
    """wall_heat_flux on the device (driver.py:132-184) from the reference's
    own padded P and from the conservative field, and the stagnation
    monitor (driver.py:187-205)."""
    from paper_2403_03440_b200 import driver
    grid, model, bcs, mech, q, cfl = golden_product(case)
    ref = get(case, f"qw_{face}")
    for src in (get(case, "P"), q):
        got = driver.wall_heat_flux(src, grid, bcs, model)
        assert set(got) == {face}
        assert got[face].shape == ref.shape
        assert np.max(np.abs(got[face] - ref)) <= 1e-12 * np.max(np.abs(ref))
    eng = driver.get_engine(grid, model)
    eng.set_bcs(bcs)
    geom = driver._WallGeom(eng, grid, bcs)
    qs = driver._stagnation_monitor_device(eng, eng.to_soa(q, eng.nv), geom)
    assert qs == pytest.approx(float(get(case, "q_stag")), rel=1e-11)


def test_wall_heat_flux_linear_profile_kat():
    """pkg/tests/test_driver.py:76-96: T linear in wall distance, the
    one-sided stencil recovers k_w * slope."""
    P = _P()
    from paper_2403_03440_b200 import driver
    from paper_2403_03440_b200.boundary import BoundaryCondition
    model = P.MixtureModel([P.SpeciesData("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0),
                            P.SpeciesData("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)])
    dims = (3, 4, 1)
    grid = P.compute_metrics(P.generate_box((0.3, 0.4, 0.1), dims))
    Tw, slope = 300.0, 500.0
    Y = np.array([0.5, 0.5])
    q = np.zeros(dims + (model.nvar,))
    for j in range(dims[1]):
        prim = P.make_primitive(model, p=1.0e5, T=Tw + slope * (j + 0.5) * 0.1, Y=Y)
        q[:, j, :, :] = P.prim_to_cons(prim, model)
    inf = P.make_primitive(model, p=1.0e5, T=Tw + slope * 0.05, Y=Y)
    bcs = {f: BoundaryCondition("farfield", freestream=inf) for f in driver.FACE_NAMES}
    bcs["jmin"] = BoundaryCondition("noslip_isothermal", T_wall=Tw)
    qw = driver.wall_heat_flux(q, grid, bcs, model)
    th = O.Thermo(model.M, model.cp_s, model.hf_s, model.Tref_s,
                  [1.663e-5, 1.919e-5], [273.15, 273.15], [107.0, 139.0])
    mu, k, _ = O.transport(np.array(Tw), Y, np.array(1.0), th)
    np.testing.assert_allclose(qw["jmin"], float(k) * slope, rtol=1e-12)
    bcs["jmin"] = BoundaryCondition("farfield", freestream=inf)
    with pytest.raises(P.NoWallBoundary):
        driver.wall_heat_flux(q, grid, bcs, model)


# ------------------------------------------------------------- f3: dual time

def _dual_case():
    from paper_2403_03440_b200.driver import Case
    grid, model, bcs, mech, q, cfl = golden_product("dual")
    v = get("dual", "bc_fs")[0]
    fr = _P().make_primitive(model, rho=v[0], u=v[1:4], T=v[4], Y=v[5:])
    return grid, model, bcs, q, fr, Case


def test_dual_time_rhs_matches_reference():
    from paper_2403_03440_b200 import implicit, spatial
    grid, model, bcs, q, fr, Case = _dual_case()
    R = spatial.assemble_residual(q, grid, bcs, None, model)
    theta, dt = get("dual", "theta_dt")
    qn, qnm1 = get("dual", "q_n"), get("dual", "q_nm1")
    got = implicit.dual_time_rhs(R, q, qn, qnm1, theta, dt, grid.volume)
    assert comp_relerr(got, get("dual", "rhs")) <= 1e-12
    got0 = implicit.dual_time_rhs(R, q, qn, qnm1, 0.0, dt, grid.volume)
    assert comp_relerr(got0, get("dual", "rhs_theta0")) <= 1e-12
    # reference KATs (test_implicit.py:290-303)
    rng = np.random.default_rng(15)
    shape = (3, 2, 1, model.nvar)
    qq = rng.random(shape) + 1.0
    vol = np.ones(shape[:3])
    np.testing.assert_array_equal(implicit.dual_time_rhs(np.zeros(shape), qq, qq, qq, 2.0, 0.1, vol),
                                  0.0)
    Rr = rng.standard_normal(shape)
    qm = qq + 0.05 * (-Rr) / vol[..., None]
    np.testing.assert_allclose(implicit.dual_time_rhs(Rr, qm, qq, qq, 0.0, 0.05, vol), 0.0,
                               atol=1e-12 * np.max(np.abs(Rr)))
    np.testing.assert_array_equal(implicit.dual_time_rhs(Rr, qm, qq, qq, 0.0, None, vol), -Rr)


@pytest.mark.parametrize("scheme", ["CS1", "CI"])
def test_dual_time_implicit_step_matches_reference(scheme):
    from paper_2403_03440_b200 import driver, spatial
    grid, model, bcs, q, fr, Case = _dual_case()
    R = spatial.assemble_residual(q, grid, bcs, None, model)
    theta, dt = get("dual", "theta_dt")
    case = Case(grid=grid, model=model, bcs=bcs, freestream=fr, scheme=scheme, cfl=5.0)
    qn, _ = driver._implicit_step(case, q, R, 5.0, theta, dt, get("dual", "q_n"), get("dual", "q_nm1"))
    ref = get("dual", f"{scheme}/q_new")
    assert comp_relerr(qn - q, ref - q) <= 1e-10


def test_unsteady_solve_matches_reference():
    """unsteady_solve (driver.py:320-359): 3 physical steps, first-order
    start, 6 inner iterations each: snapshots, times and inner residuals."""
    from paper_2403_03440_b200 import driver
    grid, model, bcs, q, fr, Case = _dual_case()
    case = Case(grid=grid, model=model, bcs=bcs, freestream=fr, scheme="CS1", cfl=5.0, dt=2e-6,
                theta=2.0, n_steps=3, inner_max=6, inner_orders=3.0)
    snaps, times, hist = driver.unsteady_solve(case, q0=q)
    ref = get("dual", "snapshots")
    assert len(snaps) == len(ref)
    np.testing.assert_allclose(times, get("dual", "times"), rtol=0, atol=0)
    for k in range(1, len(ref)):
        assert comp_relerr(snaps[k] - ref[0], ref[k] - ref[0]) <= 1e-9, k
    got, want = np.asarray(hist.res_flow), get("dual", "inner_res")
    assert got.shape == want.shape
    assert np.max(np.abs(np.log10(got) - np.log10(want))) <= 1e-9


def test_unsteady_uniform_state_is_fixed_point():
    """pkg/tests/test_driver.py:147-160: a uniform freestream box stays put."""
    P = _P()
    from paper_2403_03440_b200 import driver
    from paper_2403_03440_b200.boundary import BoundaryCondition
    model = P.MixtureModel([P.SpeciesData("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0),
                            P.SpeciesData("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)])
    grid = P.compute_metrics(P.generate_box(1.0, (4, 3, 2)))
    inf = P.make_primitive(model, rho=1.0, u=(50.0, 20.0, -30.0), T=300.0, Y=[0.6, 0.4])
    bcs = {f: BoundaryCondition("farfield", freestream=inf) for f in driver.FACE_NAMES}
    case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=inf, scheme="CS1", dt=1e-4,
                       n_steps=10, theta=2.0)
    snaps, times, hist = driver.unsteady_solve(case)
    assert len(snaps) == 11
    assert times[-1] == pytest.approx(10 * case.dt)
    q0 = snaps[0]
    for s in snaps[1:]:
        assert np.max(np.abs(s - q0)) <= 1e-10 * np.max(np.abs(q0))
    with pytest.raises(ValueError):
        driver.unsteady_solve(driver.Case(grid=grid, model=model, bcs=bcs, freestream=inf))
