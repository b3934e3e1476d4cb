"""GPU parity: the CUDA path (through the drop-in API and the C ABI) against
the reference's golden fixtures and the pinned CPU oracle.

Tolerance (north_star / SURVEY §8(d)): per component,
max_cells |X_gpu - X_ref| / max_cells |X_ref| <= 1e-10 for R, dtau, d,
lambda_face, dq*, dq and Q^{m+1} with frozen chemistry; with chemistry the
finite-difference dOmega is injected and dOmega itself is
checked against an FD-noise bound.
"""

import numpy as np
import pytest

import oracle as O
from golden_cases import comp_relerr, get, has, load, relerr
from product_cases import golden_product, spec_oracle, spec_product

pytestmark = pytest.mark.gpu

TOL = 1e-10
CASES = ["box_air5", "ogrid_air11", "chem3d", "thin", "warped"]


def _keys(case):
    return sorted({k.split("/")[1] for k in load() if k.startswith(case + "/") and k.endswith("/dq")})


CASE_KEYS = [(c, k) for c in CASES for k in _keys(c)]


def _api():
    from paper_2403_03440_b200 import driver, implicit, lusgs, spatial
    return spatial, implicit, lusgs, driver


@pytest.mark.parametrize("case", CASES)
def test_residual_matches_reference(case):
    spatial, *_ = _api()
    grid, model, bcs, mech, q, _ = golden_product(case)
    fo = bool(get(case, "first_order"))
    R, P = spatial.assemble_residual(q, grid, bcs, mech, model, first_order=fo, return_padded=True)
    assert comp_relerr(R, get(case, "R")) <= TOL
    Pref = get(case, "P")
    np.testing.assert_array_equal(np.isnan(P), np.isnan(Pref))
    assert relerr(np.nan_to_num(P), np.nan_to_num(Pref)) <= 1e-13
    R1 = spatial.assemble_residual(q, grid, bcs, mech, model, first_order=True)
    assert comp_relerr(R1, get(case, "R_first_order")) <= TOL


@pytest.mark.parametrize("case", CASES)
def test_radii_and_dtau_match_reference(case):
    _, implicit, _, _ = _api()
    from paper_2403_03440_b200.mixture import cons_to_prim
    grid, model, bcs, mech, q, cfl = golden_product(case)
    prim = cons_to_prim(q, model)
    li, lv = implicit.cell_spectral_radii(prim, grid, model)
    assert relerr(li, get(case, "lam_inv")) <= TOL
    assert relerr(lv, get(case, "lam_vis")) <= TOL
    dom = get(case, "dOm") if has(case, "dOm") else None
    dtau = implicit.pseudo_time_step(q, grid, mech, model, cfl, dom_override=dom)
    assert relerr(dtau, get(case, "dtau")) <= TOL


@pytest.mark.parametrize("case,key", CASE_KEYS)
def test_operator_sweeps_update_match_reference(case, key):
    _, implicit, lusgs, driver = _api()
    grid, model, bcs, mech, q, cfl = golden_product(case)
    scheme = key.split("_")[0]
    offd = "paper" if key.endswith("_paper") else "symmetrized"
    dom = get(case, "dOm") if has(case, "dOm") else None
    op = implicit.assemble_lhs(q, grid, scheme, get(case, "dtau"), mech, model,
                               species_offdiag=offd, dom_override=dom)
    pre = key + "/"
    assert relerr(op.w, get(case, pre + "w")) <= TOL
    assert relerr(op.b, get(case, pre + "b")) <= TOL
    assert relerr(op.d_scal, get(case, pre + "d_scal")) <= TOL
    for d in range(3):
        assert relerr(op.lam_face[d], get(case, pre + f"lam_face{d}")) <= TOL
    if scheme != "CI":
        assert relerr(op.d_species, get(case, pre + "d_species")) <= TOL
        assert relerr(op.sp_lower, get(case, pre + "sp_lower")) <= TOL
        assert relerr(op.sp_upper, get(case, pre + "sp_upper")) <= TOL
        for d in range(3):
            assert relerr(op.lam_face_sp[d], get(case, pre + f"lam_face_sp{d}")) <= TOL
    if has(case, pre + "dinv"):
        assert relerr(op.dinv_species_block, get(case, pre + "dinv")) <= 1e-9
    rhs = -get(case, "R")
    dq, star = lusgs.lusgs_solve(op, rhs, return_forward=True)
    assert comp_relerr(star, get(case, pre + "dq_star")) <= TOL
    assert comp_relerr(dq, get(case, pre + "dq")) <= TOL
    if offd == "symmetrized":
        from paper_2403_03440_b200.driver import Case
        case_obj = Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=scheme,
                        cfl=cfl)
        qn, flags, cnt, cell = driver.implicit_step_raw(case_obj, q, get(case, "R"), cfl,
                                                        dom_override=dom)
        assert comp_relerr(qn, get(case, pre + "q_new")) <= TOL
        bad = get(case, pre + "gate_bad")
        assert cnt == int(bad.sum())
        if cnt:
            assert cell == int(np.flatnonzero(bad.ravel())[0])


def test_chemistry_against_reference():
    from paper_2403_03440_b200.chemistry import production_rates, source_jacobian
    from paper_2403_03440_b200.mixture import cons_to_prim
    from product_cases import model_from_table
    from golden_cases import mech as omech
    import product_cases as pc
    model = model_from_table(get("rates", "species"), get("rates", "PrSc"))
    _, _, _, mech, q, _ = golden_product("rates")
    prim = cons_to_prim(q, model)
    om = production_rates(prim, mech, model)
    ref = get("rates", "omega")
    assert relerr(om, ref) <= 1e-12
    dOm = source_jacobian(prim, mech, model)
    dref = get("rates", "dOm")
    # FD noise bound: ulp noise in omega / h
    rho = np.asarray(prim.rho)
    h = 1e-8 * np.abs(np.asarray(prim.Y) * rho[..., None])
    h = np.maximum(h, 1e-12 * rho[..., None])
    bound = 64 * np.finfo(float).eps * np.max(np.abs(ref), axis=-1)[..., None, None] / h[..., None, :]
    assert np.all(np.abs(dOm - dref) <= bound + 1e-9 * np.abs(dref))


# ---------------------------------------------------------------- configs vs oracle

def _full_iteration_vs_oracle(spec, schemes, tol=TOL):
    from paper_2403_03440_b200 import driver, implicit, spatial
    grid, model, bcs, mech = spec_product(spec)
    th, og, obcs, omech = spec_oracle(spec)
    q = spec.q
    R = spatial.assemble_residual(q, grid, bcs, mech, model)
    Ro = O.residual(q, og, obcs, omech, th)
    assert comp_relerr(R, Ro) <= tol
    dtau = implicit.pseudo_time_step(q, grid, mech, model, spec.cfl)
    for sch in schemes:
        res = O.implicit_step(q, Ro, og, omech, th, sch, spec.cfl, want_star=False)
        assert relerr(dtau, res.dtau) <= tol
        case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=sch,
                           cfl=spec.cfl)
        qn, flags, cnt, cell = driver.implicit_step_raw(case, q, Ro, spec.cfl)
        assert comp_relerr(qn - q, res.q_new - q) <= tol
        assert cnt == int(res.bad.sum())


def test_config0_one_iteration_vs_oracle():
    from paper_2403_03440_b200 import configs as C
    _full_iteration_vs_oracle(C.config0(seed=0), ("CS1", "CS2", "CI"))


def test_config1_shape_vs_oracle():
    from paper_2403_03440_b200 import configs as C
    _full_iteration_vs_oracle(C.config1(seed=1, dims=(160, 128, 1)), ("CS1", "CI"))


def test_config2_shape_vs_oracle():
    from paper_2403_03440_b200 import configs as C
    _full_iteration_vs_oracle(C.config2(seed=2, dims=(96, 64, 1)), ("CS1",))


def test_config3_species_vs_oracle():
    from paper_2403_03440_b200 import configs as C
    for ns in (11, 20):
        _full_iteration_vs_oracle(C.config3(ns, dims=(40, 32, 1)), ("CS1", "CI"))


# ---------------------------------------------------------------- 2-D wavefront path

def _wave_vs_generic(spec, scheme, tol=1e-10):
    from paper_2403_03440_b200 import driver, spatial
    from paper_2403_03440_b200.configs import build_case
    grid, model, bcs, mech = build_case(spec)
    R = spatial.assemble_residual(spec.q, grid, bcs, mech, model)
    case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=scheme,
                       cfl=spec.cfl)
    qg, fg, cg, _, dg = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=1, want_dq=True)
    qw, fw, cw, _, dw = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=2, want_dq=True)
    assert comp_relerr(dw, dg) <= tol
    assert comp_relerr(qw - spec.q, qg - spec.q) <= tol
    assert (fw, cw) == (fg, cg)


@pytest.mark.parametrize("dims", [(64, 64, 1), (40, 45, 1), (3, 70, 1), (50, 7, 1), (33, 96, 1), (24, 330, 1)])
@pytest.mark.parametrize("scheme", ["CS1", "CS2", "CI"])
def test_wavefront_matches_generic_box(dims, scheme):
    from paper_2403_03440_b200 import configs as C
    _wave_vs_generic(C.config0(seed=7, dims=dims), scheme)


def test_wavefront_matches_generic_ogrid_and_chemistry():
    from paper_2403_03440_b200 import configs as C
    _wave_vs_generic(C.config2(seed=2, dims=(48, 40, 1)), "CS1")
    _wave_vs_generic(C.config3(20, dims=(24, 40, 1), chemistry=True), "CS1")
    _wave_vs_generic(C.config3(40, dims=(24, 36, 1)), "CS2")
    # the coupled operator on the wavefront (frozen, ns <= 16)
    _wave_vs_generic(C.config2(seed=2, dims=(48, 40, 1)), "CI")
    _wave_vs_generic(C.config3(11, dims=(40, 70, 1)), "CI")
    # large species counts: smem-resident coupled chain
    _wave_vs_generic(C.config3(20, dims=(24, 40, 1)), "CI")
    _wave_vs_generic(C.config3(40, dims=(30, 70, 1)), "CI")


def test_wavefront_nonplanar_matches_generic():
    """w != 0 on a 2-D grid (outflow k boundaries): the flow chains take the
    full 5-component path (the planar path is skipped when any z-momentum or
    its residual is nonzero)."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config0(seed=11, dims=(40, 70, 1))
    spec.bcs["kmin"] = C.BCSpec("supersonic_outflow")
    spec.bcs["kmax"] = C.BCSpec("supersonic_outflow")
    rng = np.random.default_rng(5)
    rho = spec.q[..., 0]
    w = rng.uniform(-300.0, 300.0, rho.shape)
    spec.q[..., 3] = rho * w
    spec.q[..., 4] += 0.5 * rho * w * w
    for scheme in ("CS1", "CI"):
        _wave_vs_generic(spec, scheme)


# ---------------------------------------------------------------- fused iteration (bench path)

@pytest.mark.parametrize("dims,ns", [((96, 80, 1), 5), ((33, 70, 1), 5), ((40, 66, 1), 20)])
def test_fused_iteration_matches_stages_and_oracle(dims, ns):
    """csb_iteration (residual with fused norms + implicit step, the bench's
    per-step call) against the separate stage entry points and the oracle's
    residual_norms (driver.py:85-90)."""
    import ctypes

    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.configs import build_case
    from paper_2403_03440_b200.device import SCHEMES, get_engine
    from paper_2403_03440_b200.driver import residual_norms

    # ns = 20: the species-streaming residual (NSB > 12) with fused norms
    spec = C.config0(seed=5, dims=dims) if ns == 5 else C.config3(ns, seed=5, dims=dims)
    grid, model, bcs, mech = build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    q = eng.to_soa(spec.q, eng.nv)
    qn, R, n3 = eng.empty(eng.nv, eng.N), eng.empty(eng.nv, eng.N), eng.empty(4)
    st = ctypes.c_void_p(eng.stream)
    for _ in range(3):  # repeated launches: the last-block counter must reset
        rc = eng.lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), SCHEMES["CS1"], 0, 0,
                                   qn.data_ptr(), R.data_ptr(), n3.data_ptr(), st)
        assert rc == 0, eng.lib.csb_last_error(eng.ctx)
        eng.status()
    n_fused = n3.cpu().numpy()[:3]
    Raos = eng.from_soa(R, spec.q, spec.q.shape)
    ref = residual_norms(Raos)
    n_sep = np.array([ref.flow, ref.species, ref.density])
    assert np.max(np.abs(n_fused - n_sep) / np.abs(n_sep)) <= 1e-12
    th, og, obcs, omech = spec_oracle(spec)
    on = np.array(O.norms(O.residual(spec.q, og, obcs, omech, th)))
    assert np.max(np.abs(n_fused - on) / np.abs(on)) <= 1e-10


# ---------------------------------------------------------------- steady march (driver)

def _march_case(name):
    from paper_2403_03440_b200.driver import Case
    from paper_2403_03440_b200.mixture import make_primitive
    grid, model, bcs, mech, q0, cfl = golden_product(name)
    Y = np.full(2, 0.5)
    chill = make_primitive(model, rho=1.0, T=250.0, Y=Y)
    inf = make_primitive(model, rho=1.0, T=250.0, u=(2.0 * float(chill.c), 0.0, 0.0), Y=Y)
    ramp = tuple(float(v) for v in get(name, "ramp"))
    case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, mech=mech, scheme=name[6:],
                cfl=20.0, cfl_ramp=(ramp[0], ramp[1], int(ramp[2])), max_iters=60,
                residual_drop_orders=np.inf, stop_on_absolute_floor=False)
    return case, q0


@pytest.mark.parametrize("name", ["march_CS1", "march_CI"])
def test_steady_march_matches_reference_history(name):
    """steady_solve (driver.py:266-317) over the reference's cylinder case
    (test_driver.py:108-123, 60 iterations with the CFL ramp): residual
    histories to plotting precision, CFL schedule exactly, final state."""
    from paper_2403_03440_b200.driver import steady_solve
    case, q0 = _march_case(name)
    q, hist = steady_solve(case, q0)
    assert hist.reason == "max_iters" and len(hist.iters) == 60
    assert np.array_equal(np.asarray(hist.cfl), get(name, "cfl_used"))
    for key in ("res_flow", "res_species", "res_density"):
        got, ref = np.asarray(getattr(hist, key)), get(name, key)
        assert got.shape == ref.shape
        assert np.max(np.abs(np.log10(got) - np.log10(ref))) <= 1e-9, key
    assert comp_relerr(q, get(name, "q_final")) <= 1e-9
    # stagnation heat-flux monitor samples (device wall flux, driver.py:187-205)
    got_qs, ref_qs = np.asarray(hist.q_stag, float), get(name, "q_stag_hist")
    assert np.array_equal(np.isnan(got_qs), np.isnan(ref_qs))
    m = ~np.isnan(ref_qs)
    assert m.sum() >= 6
    assert np.max(np.abs(got_qs[m] - ref_qs[m]) / np.abs(ref_qs[m])) <= 1e-9


def test_config4_reduced_march_matches_reference_history():
    """Config 4 on a reduced 48x32 O-grid (11 species, freestream start, CFL
    ramp, 40 iterations) against the reference's own steady_solve: the CFL
    halvings/recoveries and the residual histories."""
    from paper_2403_03440_b200.driver import Case, steady_solve
    from paper_2403_03440_b200.mixture import make_primitive
    name = "march_c4"
    grid, model, bcs, mech, q0, cfl = golden_product(name)
    f = get(name, "fs_prim")
    inf = make_primitive(model, rho=f[0], u=f[1:4], T=f[4], Y=f[5:])
    ramp = tuple(float(v) for v in get(name, "ramp"))
    case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, mech=mech, scheme="CS1",
                cfl=1000.0, cfl_ramp=(ramp[0], ramp[1], int(ramp[2])), max_iters=40,
                residual_drop_orders=np.inf, stop_on_absolute_floor=False)
    q, hist = steady_solve(case, q0)
    assert len(hist.iters) == 40
    np.testing.assert_allclose(np.asarray(hist.cfl), get(name, "cfl_used"), rtol=1e-12)
    for key in ("res_flow", "res_species", "res_density"):
        got, ref = np.asarray(getattr(hist, key)), get(name, key)
        assert np.max(np.abs(np.log10(got) - np.log10(ref))) <= 1e-8, key
    assert comp_relerr(q, get(name, "q_final")) <= 1e-8
