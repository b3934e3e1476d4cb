"""The reference's own known-answer tests for this path,
run against the CUDA implementation through the drop-in API.

Sources: pkg/tests/test_implicit.py (dtau examples 48-57, CS species
diagonal 145-157, LU-SGS = dense factored solve 160-187, explicit limit
190-203, reversal symmetry 206-236, corrections 239-287),
pkg/tests/test_spatial.py (freestream preservation 156-172, telescoping
175-188, first-order contact 191-223, reactor rows 226-241) and
pkg/tests/test_driver.py (fixed point 40-50, norms 53-66).
"""

import numpy as np
import pytest

from dense_operator import dense_factored_matrix

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2403_03440_b200 as P
    from paper_2403_03440_b200 import chemistry, driver, implicit, lusgs, spatial
    from paper_2403_03440_b200.boundary import BoundaryCondition
    return P, spatial, implicit, lusgs, driver, chemistry, BoundaryCondition


def binary_model():
    from paper_2403_03440_b200.mixture import MixtureModel, SpeciesData
    a = SpeciesData("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0)
    b = SpeciesData("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)
    return MixtureModel(species=(a, b), Pr=0.72, Sc=0.7)


def air5_model():
    from paper_2403_03440_b200.mixture import MixtureModel, SpeciesData
    mk = lambda n, M, cp, hf: SpeciesData(n, M, cp, hf, 298.15, 1.7e-5, 273.15, 110.0)
    return MixtureModel(species=(mk("N2", 0.0280134, 1039.0, 0.0), mk("O2", 0.0319988, 918.0, 0.0),
                                 mk("NO", 0.0300061, 995.0, 3.0e6), mk("N", 0.0140067, 1484.0, 3.36e7),
                                 mk("O", 0.0159994, 1300.0, 1.54e7)), Pr=0.72, Sc=0.7)


def all_faces(bc):
    return {n: bc for n in ("imin", "imax", "jmin", "jmax", "kmin", "kmax")}


def test_local_time_step_examples():
    P, spatial, implicit, *_ = _pkg()
    li = np.array([400.0, 0.0, 0.0])
    assert implicit.local_time_step(li, np.zeros(3), 0.0, 5.0, 1.0) == pytest.approx(0.0125, rel=1e-14)
    assert implicit.local_time_step(li, np.zeros(3), 0.0, 10.0, 1.0) == pytest.approx(0.025)
    assert implicit.local_time_step(li, np.zeros(3), 1200.0, 5.0, 1.0) == pytest.approx(0.0125 / 4, rel=1e-14)
    with pytest.raises(P.ZeroWavespeed):
        implicit.local_time_step(np.zeros(3), np.zeros(3), 0.0, 5.0, 1.0)


def test_cs_species_diag_example():
    P, spatial, implicit, *_ = _pkg()
    from paper_2403_03440_b200.mixture import MixtureModel, SpeciesData
    mk = lambda n: SpeciesData(n, 0.028, 1039.0, 0.0, 0.0, 0.0, 273.15, 107.0)
    model = MixtureModel(species=(mk("A"), mk("B")), Pr=0.72, Sc=0.7)
    grid = P.compute_metrics(P.generate_box((2.0, 1.0, 1.0), (2, 1, 1)))
    inf = P.make_primitive(model, rho=1.0, u=(100.0, 0.0, 0.0), T=300.0, Y=[0.5, 0.5])
    q = np.broadcast_to(P.prim_to_cons(inf, model), (2, 1, 1, model.nvar)).copy()
    op = implicit.assemble_lhs(q, grid, "CS1", 0.01, None, model)
    np.testing.assert_allclose(op.d_species[0, 0, 0], 200.0, rtol=1e-12)


def _uniform_operator(model, mode, dims=(4, 4, 1), cfl=5.0, mech=None, seed=None,
                      species_offdiag="symmetrized"):
    P, spatial, implicit, *_ = _pkg()
    from paper_2403_03440_b200.chemistry import source_jacobian, source_spectral_radius
    grid = P.compute_metrics(P.generate_box(1.0, dims))
    Y = np.full(model.ns, 1.0 / model.ns)
    inf = P.make_primitive(model, rho=1.0, u=(150.0, 40.0, 0.0), T=400.0, Y=Y)
    q = np.broadcast_to(P.prim_to_cons(inf, model), dims + (model.nvar,)).copy()
    if seed is not None:
        q *= 1.0 + 0.05 * np.random.default_rng(seed).random(q.shape)
    prim = P.cons_to_prim(q, model)
    li, lv = implicit.cell_spectral_radii(prim, grid, model)
    lS = source_spectral_radius(source_jacobian(prim, mech, model)) if mech else 0.0
    dtau = implicit.local_time_step(li, lv, lS, cfl, grid.J)
    return grid, q, implicit.assemble_lhs(q, grid, mode, dtau, mech, model,
                                          species_offdiag=species_offdiag)


@pytest.mark.parametrize("mode", ["CI", "CS1", "CS2"])
@pytest.mark.parametrize("with_chem", [False, True])
def test_lusgs_matches_dense_factored_solve(mode, with_chem):
    P, spatial, implicit, lusgs, driver, chemistry, _ = _pkg()
    model = binary_model()
    mech = None
    if with_chem:
        mech = chemistry.Mechanism(reactions=(chemistry.Reaction(
            np.array([1.0, 0.0]), np.array([0.0, 1.0]), A_f=20.0, b_f=0.0, Ea_f=0.0,
            backward=(10.0, 0.0, 0.0)),))
    grid, q, op = _uniform_operator(model, mode, mech=mech, seed=5)
    rhs = np.random.default_rng(6).standard_normal(q.shape) * 100.0
    dq = lusgs.lusgs_solve(op, rhs)
    expect = np.linalg.solve(dense_factored_matrix(op, grid), rhs.reshape(-1)).reshape(q.shape)
    np.testing.assert_allclose(dq, expect, atol=1e-12 * np.max(np.abs(expect)))


@pytest.mark.parametrize("mode", ["CI", "CS1"])
def test_lusgs_paper_offdiag_variant_matches_dense(mode):
    P, spatial, implicit, lusgs, *_ = _pkg()
    grid, q, op = _uniform_operator(binary_model(), mode, dims=(3, 2, 2), seed=8,
                                    species_offdiag="paper")
    rhs = np.random.default_rng(9).standard_normal(q.shape)
    dq = lusgs.lusgs_solve(op, rhs)
    expect = np.linalg.solve(dense_factored_matrix(op, grid), rhs.reshape(-1)).reshape(q.shape)
    np.testing.assert_allclose(dq, expect, atol=1e-12 * np.max(np.abs(expect)))


def test_lusgs_diagonal_system():
    P, spatial, implicit, lusgs, *_ = _pkg()
    model = binary_model()
    grid = P.compute_metrics(P.generate_box(1.0, (3, 3, 2)))
    inf = P.make_primitive(model, rho=1.0, u=(100.0, 0.0, 0.0), T=300.0, Y=[0.5, 0.5])
    q = np.broadcast_to(P.prim_to_cons(inf, model), grid.dims + (model.nvar,)).copy()
    dtau = np.full(grid.dims, 1e-17)
    op = implicit.assemble_lhs(q, grid, "CI", dtau, None, model)
    rhs = np.random.default_rng(10).standard_normal(q.shape)
    dq = lusgs.lusgs_solve(op, rhs)
    expect = grid.J[..., None] * dtau[..., None] * rhs
    assert np.max(np.abs(dq - expect)) <= 1e-8 * np.max(np.abs(expect))


def test_lusgs_reversal_symmetry():
    P, spatial, implicit, lusgs, *_ = _pkg()
    from paper_2403_03440_b200.mixture import MixtureModel, SpeciesData
    model = MixtureModel(species=(SpeciesData("A", 0.028, 1039.0, 0.0, 0.0, 0.0, 273.15, 107.0),
                                  SpeciesData("B", 0.032, 918.0, 0.0, 0.0, 0.0, 273.15, 107.0)),
                         Pr=0.72, Sc=0.7)
    dims = (8, 1, 1)
    grid = P.compute_metrics(P.generate_box((1.0, 0.2, 0.2), dims))
    pf = P.make_primitive(model, rho=1.1, u=(80.0, 0.0, 0.0), T=300.0, Y=[0.4, 0.6])
    pb = P.make_primitive(model, rho=1.1, u=(-80.0, 0.0, 0.0), T=300.0, Y=[0.4, 0.6])
    qf = np.zeros(dims + (model.nvar,))
    qb = np.zeros_like(qf)
    qf[..., :] = P.prim_to_cons(pf, model)
    qb[..., :] = P.prim_to_cons(pb, model)
    op_f = implicit.assemble_lhs(qf, grid, "CS1", 1e-3, None, model)
    rhs = np.zeros(qf.shape)
    rhs[..., 5:] = np.random.default_rng(12).standard_normal(rhs[..., 5:].shape)
    dq_f = lusgs.lusgs_solve(op_f, rhs)
    op_b = implicit.assemble_lhs(qb, grid, "CS1", 1e-3, None, model)
    dq_b = lusgs.lusgs_solve(op_b, rhs[::-1].copy())
    np.testing.assert_allclose(dq_f, dq_b[::-1], atol=1e-12 * np.max(np.abs(dq_f)))
    np.testing.assert_array_equal(dq_f[..., :5], 0.0)


def test_corrections_hand_values_and_fixed_points():
    P, spatial, implicit, *_ = _pkg()
    out = implicit.correct_increment_cs1(np.array([0.5, 0.5]), np.array([0.06, 0.03]), 0.1)
    np.testing.assert_allclose(out, [0.565, 0.535], rtol=1e-15)
    out = implicit.correct_normalize_cs2(np.array([0.5, 0.5]), np.array([0.06, 0.03]), 0.1)
    np.testing.assert_allclose(out, [0.5651376146788991, 0.534862385321101], rtol=1e-15)
    rs = np.array([0.3, 0.7])
    np.testing.assert_allclose(implicit.correct_increment_cs1(rs, np.array([0.02, 0.05]), 0.07),
                               rs + [0.02, 0.05], rtol=1e-15)
    np.testing.assert_array_equal(implicit.correct_increment_cs1(rs, np.zeros(2), 0.0), rs)
    np.testing.assert_allclose(implicit.correct_normalize_cs2(np.array([1.2]), np.array([0.1]), 0.1),
                               [1.3], rtol=1e-15)
    with pytest.raises(P.NonPhysicalState):
        implicit.correct_increment_cs1(np.array([1e-6, 1.0]), np.array([-1e-3, 0.0]), -1e-3)


def test_corrections_no_drift_many_rows():
    P, spatial, implicit, *_ = _pkg()
    rng = np.random.default_rng(14)
    r1 = np.tile(np.array([0.2, 0.5, 0.3]), (64, 1))
    r2 = r1.copy()
    for _ in range(200):
        d = 1e-4 * rng.standard_normal(r1.shape)
        drho = d.sum(-1) + 1e-5 * rng.standard_normal(64)
        r1 = implicit.correct_increment_cs1(r1, d, drho)
        r2 = implicit.correct_normalize_cs2(r2, d, drho)
        for r in (r1, r2):
            assert np.max(np.abs((r / r.sum(-1, keepdims=True)).sum(-1) - 1.0)) <= 1e-12


@pytest.mark.parametrize("gridder", ["box", "warped", "ogrid"])
def test_freestream_preservation(gridder):
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = air5_model()
    if gridder == "box":
        nodes = P.generate_box(1.0, (6, 5, 4))
    elif gridder == "warped":
        nodes = P.generate_box(1.0, (6, 5, 4))
        nodes[1:-1, 1:-1, 1:-1] += 0.02 * np.random.default_rng(12).standard_normal(
            nodes[1:-1, 1:-1, 1:-1].shape)
    else:
        nodes = P.generate_cylinder_ogrid(0.045, 0.3, (12, 10, 1), stretch=1.1)
    grid = P.compute_metrics(nodes)
    inf = P.make_primitive(model, rho=0.8, u=(220.0, -45.0, 10.0), T=500.0,
                           Y=[0.7, 0.2, 0.05, 0.03, 0.02])
    q0 = P.prim_to_cons(inf, model)
    q = np.broadcast_to(q0, grid.dims + (model.nvar,)).copy()
    R = spatial.assemble_residual(q, grid, all_faces(BC("farfield", freestream=inf)), None, model)
    scale = 0.0  # flux_scale (test_spatial.py:34-36)
    for d in range(3):
        S = grid.face_areas(d)
        U = np.einsum("...c,c->...", S, np.asarray(inf.u))
        F = U[..., None] * q0
        F[..., 1:4] += float(inf.p) * S
        F[..., 4] += float(inf.p) * U
        scale = max(scale, float(np.max(np.abs(F))))
    assert np.max(np.abs(R)) <= 1e-12 * scale


def test_conservation_telescoping():
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = binary_model()
    grid = P.compute_metrics(P.generate_box(1.0, (4, 4, 4)))
    inf = P.make_primitive(model, rho=1.0, u=(50.0, 20.0, -30.0), T=300.0, Y=[0.6, 0.4])
    q = np.broadcast_to(P.prim_to_cons(inf, model), grid.dims + (model.nvar,)).copy()
    q *= 1.0 + 0.01 * np.random.default_rng(3).standard_normal(q.shape)
    R = spatial.assemble_residual(q, grid, all_faces(BC("periodic")), None, model)
    q0 = P.prim_to_cons(inf, model)
    scale = np.max(np.abs(q0)) * 400.0
    np.testing.assert_allclose(R.sum(axis=(0, 1, 2)), 0.0, atol=1e-12 * scale)


def test_reactor_source_rows():
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = binary_model()
    mech = chemistry.Mechanism(reactions=(chemistry.Reaction(np.array([1.0, 0.0]), np.array([0.0, 1.0]),
                                                             A_f=5.0, b_f=0.0, Ea_f=0.0),))
    grid = P.compute_metrics(P.generate_box(1.0, (3, 3, 1)))
    prim = P.make_primitive(model, rho=1.0, u=(25.0, 0.0, 0.0), T=400.0, Y=[0.5, 0.5])
    q = np.broadcast_to(P.prim_to_cons(prim, model), grid.dims + (model.nvar,)).copy()
    R = spatial.assemble_residual(q, grid, all_faces(BC("periodic")), mech, model)
    omega = chemistry.production_rates(P.cons_to_prim(q[0, 0, 0], model), mech, model)
    np.testing.assert_allclose(R[..., :5], 0.0, atol=1e-9)
    np.testing.assert_allclose(R[..., 5:], -omega * grid.volume[..., None], rtol=1e-12, atol=1e-20)


def test_uniform_freestream_fixed_point_over_steps():
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = binary_model()
    for scheme in ("CI", "CS1", "CS2"):
        grid = P.compute_metrics(P.generate_box(1.0, (5, 4, 3)))
        inf = P.make_primitive(model, rho=1.0, u=(180.0, -40.0, 20.0), T=300.0, Y=[0.5, 0.5])
        case = driver.Case(grid=grid, model=model, bcs=all_faces(BC("farfield", freestream=inf)),
                           freestream=inf, scheme=scheme, max_iters=50,
                           residual_drop_orders=np.inf, stop_on_absolute_floor=False)
        q0 = case.initial_field()
        q, hist = driver.steady_solve(case)
        assert hist.reason == "max_iters" and len(hist.iters) == 50
        assert np.max(np.abs(q - q0)) <= 1e-11 * np.max(np.abs(q0))


def test_residual_norm_definitions():
    P, spatial, implicit, lusgs, driver, *_ = _pkg()
    R = np.zeros((4, 3, 2, 7))
    n = driver.residual_norms(R)
    assert n.flow == n.species == n.density == 0.0
    R[..., 0] = 1.0
    n = driver.residual_norms(R)
    assert n.density == pytest.approx(np.sqrt(24)) and n.flow == pytest.approx(np.sqrt(24))
    R = np.zeros((4, 3, 2, 7))
    R[..., 5] = 0.5
    R[..., 6] = -0.2
    assert driver.residual_norms(R).species == pytest.approx(np.sqrt(24 * 0.3 ** 2))


def test_missing_bc_raises():
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = binary_model()
    grid = P.compute_metrics(P.generate_box(1.0, (4, 3, 2)))
    inf = P.make_primitive(model, rho=1.0, T=300.0, Y=[0.5, 0.5])
    q = np.broadcast_to(P.prim_to_cons(inf, model), grid.dims + (model.nvar,)).copy()
    bcs = all_faces(BC("farfield", freestream=inf))
    del bcs["jmax"]
    with pytest.raises(P.MissingBC):
        spatial.assemble_residual(q, grid, bcs, None, model)
    bcs = all_faces(BC("farfield", freestream=inf))
    bcs["imin"] = BC("periodic")
    with pytest.raises(P.MissingBC):
        spatial.assemble_residual(q, grid, bcs, None, model)


def test_nonphysical_state_raises():
    P, spatial, implicit, lusgs, driver, chemistry, BC = _pkg()
    model = binary_model()
    grid = P.compute_metrics(P.generate_box(1.0, (4, 3, 1)))
    inf = P.make_primitive(model, rho=1.0, T=300.0, Y=[0.5, 0.5])
    q = np.broadcast_to(P.prim_to_cons(inf, model), grid.dims + (model.nvar,)).copy()
    q[1, 1, 0, 0] = -1.0
    with pytest.raises(P.NonPhysicalState):
        spatial.assemble_residual(q, grid, all_faces(BC("farfield", freestream=inf)), None, model)
    with pytest.raises(P.NonPhysicalState):
        P.cons_to_prim(q, model)


@pytest.mark.gpu
@pytest.mark.parametrize("ns", [2, 5, 8, 11, 16, 20, 23, 32])
def test_species_block_inverse_matches_numpy_inv(ns):
    """csb_batched_inverse against the reference's numpy.linalg.inv of
    d I - V dOmega (implicit.py:362-368) on seeded blocks, including blocks
    that need row pivoting."""
    from paper_2403_03440_b200.implicit import species_block_inverse
    rng = np.random.default_rng(100 + ns)
    N = 1000
    dOm = rng.normal(size=(N, ns, ns))
    V = rng.uniform(0.5, 2.0, N)
    d = rng.uniform(0.1, 3.0, N) * ns
    d[:50] = 0.0  # zero diagonal: pivoting required
    blk = d[:, None, None] * np.eye(ns) - V[:, None, None] * dOm
    ref = np.linalg.inv(blk)
    got = species_block_inverse(d, V, dOm)
    cond = np.linalg.cond(blk)
    err = np.max(np.abs(got - ref), axis=(1, 2)) / np.max(np.abs(ref), axis=(1, 2))
    assert np.all(err <= 1e-13 * np.maximum(cond, 1.0)), float(np.max(err / np.maximum(cond, 1.0)))


@pytest.mark.gpu
def test_species_block_inverse_singular_raises():
    from paper_2403_03440_b200.errors import SingularDiagonal
    from paper_2403_03440_b200.implicit import species_block_inverse
    ns = 4
    dOm = np.zeros((3, ns, ns))
    with pytest.raises(SingularDiagonal):
        species_block_inverse(np.array([1.0, 0.0, 1.0]), np.ones(3), dOm)
