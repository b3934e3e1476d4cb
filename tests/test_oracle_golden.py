"""Pin the CPU oracle to the real reference's outputs (tests/golden/).

The fixtures were produced by tests/golden/make_golden.py running
/root/reference; these tests run anywhere (CPU only) and must be green
before the oracle is trusted as the GPU parity checker.
"""

import numpy as np
import pytest

import oracle as O
from golden_cases import bcs, comp_relerr, get, grid, has, mech, relerr, thermo

ONE_ITER = ["box_air5", "ogrid_air11", "chem3d", "thin", "warped"]
TOL = 1e-13


@pytest.mark.parametrize("case", ONE_ITER)
def test_metrics(case):
    g = grid(case)
    np.testing.assert_array_equal(g.volume, get(case, "vol"))
    for d, k in enumerate(("Si", "Sj", "Sk")):
        np.testing.assert_array_equal(g.S(d), get(case, k))


@pytest.mark.parametrize("case", ONE_ITER)
def test_residual_and_padded(case):
    th, g = thermo(case), grid(case)
    q = get(case, "q")
    fo = bool(get(case, "first_order"))
    R, P = O.residual(q, g, bcs(case, th), mech(case), th, first_order=fo, want_padded=True)
    Pref = get(case, "P")
    assert np.array_equal(np.isnan(P), np.isnan(Pref))
    np.testing.assert_array_equal(np.nan_to_num(P), np.nan_to_num(Pref))
    assert comp_relerr(R, get(case, "R")) <= TOL
    R1 = O.residual(q, g, bcs(case, th), mech(case), th, first_order=True)
    assert comp_relerr(R1, get(case, "R_first_order")) <= TOL
    fl, sp, de = O.norms(R)
    np.testing.assert_allclose([fl, sp, de], get(case, "norms"), rtol=1e-13)


@pytest.mark.parametrize("case", ONE_ITER)
def test_radii_dtau(case):
    th, g = thermo(case), grid(case)
    q = get(case, "q")
    pr = O.decode(q, th)
    li, lv = O.cell_radii(pr, g, th)
    assert relerr(li, get(case, "lam_inv")) <= TOL
    assert relerr(lv, get(case, "lam_vis")) <= TOL
    m = mech(case)
    lS = 0.0
    if O.chem_active(m):
        dOm = O.source_jac(pr, m, th)
        np.testing.assert_array_equal(dOm, get(case, "dOm"))
        lS = O.source_radius(dOm)
    dtau = O.time_step(li, lv, lS, float(get(case, "cfl")), g.J)
    assert relerr(dtau, get(case, "dtau")) <= TOL


def _schemes(case):
    z = [k.split("/")[1] for k in __import__("golden_cases").load() if k.startswith(case + "/")
         and k.endswith("/dq")]
    return sorted(set(z))


CASE_SCHEMES = [(c, s) for c in ONE_ITER for s in _schemes(c)]


@pytest.mark.parametrize("case,key", CASE_SCHEMES)
def test_operator_sweeps_update(case, key):
    th, g = thermo(case), grid(case)
    q = get(case, "q")
    m = mech(case)
    scheme = key.split("_")[0]
    offd = "paper" if key.endswith("_paper") else "symmetrized"
    dtau = get(case, "dtau")
    op = O.assemble(q, g, scheme, dtau, m, th, offd)
    pre = f"{key}/"
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
        assert relerr(op.dinv_blk, get(case, pre + "dinv")) <= 1e-12
    rhs = -get(case, "R")
    star = O.solve(op, rhs, g, forward_only=True)
    assert comp_relerr(star, get(case, pre + "dq_star")) <= 1e-12
    dq = O.solve(op, rhs, g)
    assert comp_relerr(dq, get(case, pre + "dq")) <= 1e-12
    qn, bad = O.update(q, get(case, pre + "dq"), scheme, th)
    assert comp_relerr(qn, get(case, pre + "q_new")) <= TOL
    np.testing.assert_array_equal(bad, get(case, pre + "gate_bad"))


def test_chemistry_rates_and_jacobian():
    th = thermo("rates")
    m = mech("rates")
    pr = O.decode(get("rates", "q"), th)
    np.testing.assert_array_equal(O.production(pr, m, th), get("rates", "omega"))
    dOm = O.source_jac(pr, m, th)
    np.testing.assert_array_equal(dOm, get("rates", "dOm"))
    np.testing.assert_array_equal(O.source_radius(dOm), get("rates", "lam_S"))


def test_full_step_chem3d_matches():
    case = "chem3d"
    th, g = thermo(case), grid(case)
    q = get(case, "q")
    R = O.residual(q, g, bcs(case, th), mech(case), th)
    res = O.implicit_step(q, R, g, mech(case), th, "CS1", float(get(case, "cfl")))
    assert comp_relerr(res.dq, get(case, "CS1/dq")) <= 1e-12
    assert comp_relerr(res.q_new, get(case, "CS1/q_new")) <= 1e-12
