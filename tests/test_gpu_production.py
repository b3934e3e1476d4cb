"""GPU parity at the production launch shapes and the stated configs.

Every case runs the CUDA path through the drop-in API / C ABI and compares
it with the pinned CPU oracle (oracle/csflow_oracle.py, itself checked
against the reference's golden fixtures) on identical seeded inputs.

Tolerance (north_star): per component,
max_cells |X_gpu - X_ref| / max_cells |X_ref| <= 1e-10 for R, dtau, dq and
Q^{m+1}; with chemistry the GPU's finite-difference dOmega is injected into
both sides and dOmega itself is checked entry by entry against
the FD-noise bound C eps max|omega| / h.

Launch shapes covered (csb_wave.cuh launch_wave_step):
  * > 24 strips: the forward sweep runs AFTER the records kernel (serial
    order, the 1024^2 and config-4 production order), and the same grid with
    CSB_FORCE_OVERLAP (records and forward sweep concurrent);
  * > 74 strips: more sweep CTAs than SMs, deadlock freedom from the ticket
    order alone;
  * the full config-1 (512^2) and config-3 (1024^2) grids.
"""

import os

import numpy as np
import pytest

import oracle as O
from golden_cases import comp_relerr, relerr
from product_cases import spec_oracle, spec_product

pytestmark = pytest.mark.gpu

TOL = 1e-10


class _env:
    """Temporarily set launcher knobs (csb_wave.cuh reads them per launch)."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = os.environ.get(k)
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _iteration(spec, schemes, *, offdiag="symmetrized", path=0, check_R=True, tol=TOL,
               chemistry=False):
    """One full implicit iteration per scheme: R, dtau, dq and Q^{m+1} (and
    the gate count) against the oracle.  Returns the per-scheme errors."""
    from paper_2403_03440_b200 import driver, implicit, spatial
    from paper_2403_03440_b200.chemistry import source_jacobian
    from paper_2403_03440_b200.mixture import cons_to_prim
    grid, model, bcs, mech = spec_product(spec)
    th, og, obcs, omech = spec_oracle(spec)
    q = spec.q
    R = spatial.assemble_residual(q, grid, bcs, mech, model)
    Ro = O.residual(q, og, obcs, omech, th)
    errs = {"R": comp_relerr(R, Ro)}
    if check_R:
        assert errs["R"] <= tol, errs
    dom = None
    if chemistry:
        dom = np.asarray(source_jacobian(cons_to_prim(q, model), mech, model))
        pr = O.decode(q, th)
        dref = O.source_jac(pr, omech, th)
        _check_dom(dom, dref, pr, omech, th)
    for sch in schemes:
        res = O.implicit_step(q, Ro, og, omech, th, sch, spec.cfl, species_offdiag=offdiag,
                              dom_override=dom, want_star=False)
        dtau = implicit.pseudo_time_step(q, grid, mech, model, spec.cfl, dom_override=dom)
        errs[f"{sch}/dtau"] = relerr(dtau, res.dtau)
        case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme=sch,
                           cfl=spec.cfl, species_offdiag=offdiag)
        qn, flags, cnt, cell, dq = driver.implicit_step_raw(case, q, Ro, spec.cfl, dom_override=dom,
                                                            path=path, want_dq=True)
        errs[f"{sch}/dq"] = comp_relerr(dq, res.dq)
        errs[f"{sch}/q_new"] = comp_relerr(qn - q, res.q_new - q)
        assert errs[f"{sch}/dtau"] <= tol, errs
        assert errs[f"{sch}/dq"] <= tol, errs
        assert errs[f"{sch}/q_new"] <= tol, errs
        assert cnt == int(res.bad.sum()), (sch, cnt, int(res.bad.sum()))
        if cnt:
            assert cell == int(np.flatnonzero(res.bad.ravel())[0])
    return errs


def _check_dom(dom, dref, pr, mech, th):
    """dOmega against the oracle's within the FD noise: the
    central difference divides ulp noise of omega by 2h."""
    rho = np.asarray(pr.rho)
    rs = rho[..., None] * pr.Y
    h = np.maximum(1e-8 * np.abs(rs), 1e-12 * rho[..., None])
    om = np.abs(O.rates(np.asarray(pr.T), rs, mech, th))
    # |omega| of the perturbed states is bounded by the sum of the magnitudes
    # of the reaction terms; max over species of |omega| is a lower bound, so
    # use the per-cell sum of |omega_s| with a generous ulp multiplier
    scale = np.sum(om, axis=-1)[..., None, None] + 1e-300
    bound = 256 * np.finfo(float).eps * scale / h[..., None, :]
    err = np.abs(dom - dref)
    assert np.all(err <= bound + 1e-9 * np.abs(dref)), float(np.max(err / (bound + 1e-9 * np.abs(dref))))


# ------------------------------------------------------- (a) launch shapes


@pytest.mark.slow
@pytest.mark.parametrize("overlap", ["serial", "forced"])
def test_26_strips_serial_and_overlapped_vs_oracle(overlap):
    """96 x 832 cells = 26 strips: 52 sweep CTAs > 48, so production runs the
    records kernel and the forward sweep serially; CSB_FORCE_OVERLAP runs
    them concurrently (records tiles published per step block)."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config0(seed=21, dims=(96, 832, 1))
    env = {"CSB_FORCE_OVERLAP": "1" if overlap == "forced" else None, "CSB_NO_OVERLAP": None}
    with _env(**env):
        _iteration(spec, ("CS1", "CS2", "CI"), path=2)


def test_75_strips_more_sweep_ctas_than_sms_vs_oracle():
    """8 x 2400 cells = 75 strips: 150 sweep CTAs on 148 SMs (CS) and 75
    coupled CTAs (CI); strips start in ticket order."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config0(seed=22, dims=(8, 2400, 1))
    _iteration(spec, ("CS1", "CI"), path=2)


def test_no_overlap_knob_small_grid_vs_oracle():
    """A 5-strip grid normally overlapped; CSB_NO_OVERLAP forces the serial order."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config0(seed=23, dims=(70, 150, 1))
    with _env(CSB_NO_OVERLAP="1"):
        _iteration(spec, ("CS1", "CI"), path=2)
    _iteration(spec, ("CS1",), path=2)


# ------------------------------------------------------- (b, c) stated configs at full size


@pytest.mark.slow
def test_config1_full_512_vs_oracle():
    """Config 1 at its stated 512 x 512 size: one CS1 and one CI iteration."""
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config1(seed=1), ("CS1", "CI"))


@pytest.mark.slow
def test_config3_ns11_full_1024_vs_oracle():
    """Config 3, ns = 11, at its stated 1024 x 1024 size: one CS1 iteration."""
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config3(11, seed=3), ("CS1",))


@pytest.mark.slow
def test_config2_full_1024_one_iteration_vs_oracle():
    """Config 2 (1024^2 O-grid, 11 species, smoothed fields, CFL 100) at its
    stated size: one CS1 iteration at function level with the gate reported
    (SURVEY G11 option (i)); the gate-failure count and first cell must match."""
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config2(seed=2), ("CS1",))


# ------------------------------------------------------- (d) ns = 40


def test_ns40_iteration_vs_oracle():
    """Bucket 40: species-streaming residual, 5 species warps, smem-resident
    coupled chain -- CS1, CS2 and CI against the oracle."""
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config3(40, seed=3, dims=(64, 96, 1)), ("CS1", "CS2", "CI"))


def test_ns20_iteration_vs_oracle():
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config3(20, seed=4, dims=(48, 70, 1)), ("CS1", "CS2", "CI"))


# ------------------------------------------------------- (e) synthetic chemistry


@pytest.mark.parametrize("ns", [20, 40])
def test_config3_synthetic_chemistry_vs_oracle(ns):
    """Config-3 synthetic mechanisms (2 ns reversible reactions, stiff
    Arrhenius data): residual with omega V, dOmega per entry against the
    FD-noise bound, then CS1 and CI with dOmega injected."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config3(ns, seed=3, dims=(24, 40, 1), chemistry=True)
    _iteration(spec, ("CS1", "CI"), chemistry=True)


@pytest.mark.parametrize("ns,rec", [(11, None), (11, "4"), (20, None), (40, None)])
def test_serial_order_chemistry_sliding_records_vs_oracle(ns, rec):
    """Serial launch order (what every grid above 24 strips runs): the
    sliding-window records kernel with per-species diagonals (dOmega) and
    lam_S, at the block length the launcher picks and at a forced one."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config3(ns, seed=5, dims=(40, 72, 1), chemistry=True)
    with _env(CSB_NO_OVERLAP="1", CSB_REC_S=rec):
        _iteration(spec, ("CS1", "CI") if ns <= 16 else ("CS1",), chemistry=True, path=2)


@pytest.mark.parametrize("rec", ["0", "4", "8", "16"])
def test_serial_order_records_block_lengths_vs_oracle(rec):
    """Every records variant of the serial order (tile kernel, 4- / 8- /
    16-step sliding blocks) on a grid with partial strips and partial chunks."""
    from paper_2403_03440_b200 import configs as C
    spec = C.config0(seed=25, dims=(150, 75, 1))
    with _env(CSB_NO_OVERLAP="1", CSB_REC_S=rec):
        _iteration(spec, ("CS1", "CS2", "CI"), path=2)


@pytest.mark.parametrize("kbc", ["supersonic_outflow", "symmetry"])
def test_residual_fallback_chain_w_nonzero_vs_oracle(kbc):
    """The planar 2-D residual (w == 0) finds w != 0: the K2D kernel re-runs on
    the device (outflow k boundaries), and under symmetry k boundaries the
    general path after it; R, the fused norms of csb_iteration and a second
    call (the context then skips the planar variant) all match the oracle."""
    import ctypes

    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200 import spatial
    from paper_2403_03440_b200.configs import build_case
    from paper_2403_03440_b200.device import SCHEMES, get_engine
    spec = C.config0(seed=31, dims=(45, 52, 1))
    spec.bcs["kmin"] = C.BCSpec(kbc)
    spec.bcs["kmax"] = C.BCSpec(kbc)
    rng = np.random.default_rng(7)
    rho = spec.q[..., 0]
    w = rng.uniform(-300.0, 300.0, rho.shape)
    spec.q[..., 3] = rho * w
    spec.q[..., 4] += 0.5 * rho * w * w
    grid, model, bcs, mech = spec_product(spec)
    th, og, obcs, omech = spec_oracle(spec)
    Ro = O.residual(spec.q, og, obcs, omech, th)
    for _ in range(2):
        R = spatial.assemble_residual(spec.q, grid, bcs, mech, model)
        assert comp_relerr(R, Ro) <= TOL
    # fused iteration entry (residual + norms + implicit step) on a fresh context
    grid2, model2, bcs2, mech2 = build_case(spec)
    eng = get_engine(grid2, model2)
    eng.set_bcs(bcs2)
    eng.set_mechanism(mech2)
    q = eng.to_soa(spec.q, eng.nv)
    qn, Rd, norms = eng.empty(eng.nv, eng.N), eng.empty(eng.nv, eng.N), eng.empty(4)
    st = ctypes.c_void_p(eng.stream)
    on = np.array(O.norms(Ro))
    for _ in range(2):  # (the second call runs with the planar variant disabled)
        rc = eng.lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), SCHEMES["CS1"], 0, 0,
                                   qn.data_ptr(), Rd.data_ptr(), norms.data_ptr(), st)
        assert rc == 0, eng.lib.csb_last_error(eng.ctx)
        eng.status()
        Rg = eng.from_soa(Rd, spec.q, spec.q.shape)
        assert comp_relerr(np.asarray(Rg), Ro) <= TOL
        got = norms.cpu().numpy()[:3]
        assert np.max(np.abs(got - on) / np.abs(on)) <= 1e-10


# ------------------------------------------------------- (f) paper species off-diagonal


@pytest.mark.parametrize("dims", [(64, 64, 1), (40, 800, 1)])
def test_wavefront_paper_offdiag_vs_oracle(dims):
    """species_offdiag = "paper" (sp_scale 1, implicit.py:385) on the 2-D
    wavefront, including a 25-strip grid."""
    from paper_2403_03440_b200 import configs as C
    _iteration(C.config0(seed=24, dims=dims), ("CS1", "CS2"), offdiag="paper", path=2)


# ------------------------------------------------------- (g) the bench's entry point


@pytest.mark.parametrize("dims,ns,scheme", [((96, 80, 1), 5, "CS1"), ((40, 810, 1), 11, "CS1"),
                                            ((40, 66, 1), 20, "CI")])
def test_csb_iteration_q_new_vs_oracle(dims, ns, scheme):
    """csb_iteration (residual + fused norms + implicit step, the bench's
    per-step call) -> Q^{m+1} and the norms against the oracle."""
    import ctypes

    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.configs import build_case
    from paper_2403_03440_b200.device import SCHEMES, get_engine
    spec = C.config0(seed=5, dims=dims) if ns == 5 else C.config3(ns, seed=5, dims=dims)
    grid, model, bcs, mech = build_case(spec)
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    q = eng.to_soa(spec.q, eng.nv)
    qn, R, n3 = eng.empty(eng.nv, eng.N), eng.empty(eng.nv, eng.N), eng.empty(4)
    st = ctypes.c_void_p(eng.stream)
    rc = eng.lib.csb_iteration(eng.ctx, q.data_ptr(), float(spec.cfl), SCHEMES[scheme], 0, 0,
                               qn.data_ptr(), R.data_ptr(), n3.data_ptr(), st)
    assert rc == 0, eng.lib.csb_last_error(eng.ctx)
    flags, cell, cnt = eng.status()
    th, og, obcs, omech = spec_oracle(spec)
    Ro = O.residual(spec.q, og, obcs, omech, th)
    res = O.implicit_step(spec.q, Ro, og, omech, th, scheme, spec.cfl, want_star=False)
    q_new = eng.from_soa(qn, spec.q, spec.q.shape)
    assert comp_relerr(eng.from_soa(R, spec.q, spec.q.shape), Ro) <= TOL
    assert comp_relerr(q_new - spec.q, res.q_new - spec.q) <= TOL
    assert cnt == int(res.bad.sum())
    on = np.array(O.norms(Ro))
    assert np.max(np.abs(n3.cpu().numpy()[:3] - on) / np.abs(on)) <= 1e-10


# ------------------------------------------------------- species slot sizes


@pytest.mark.parametrize("ns", [24, 48])
def test_wavefront_chemistry_ring_fits_at_buckets_24_48(ns):
    """CS with chemistry at the widest species record layouts: the species
    ring must fit shared memory (path=2 fails loudly otherwise) and match the
    generic hyperplane sweeps."""
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200 import driver, spatial
    from paper_2403_03440_b200.configs import build_case
    spec = C.config3(ns, seed=9, dims=(20, 70, 1), chemistry=True)
    grid, model, bcs, mech = build_case(spec)
    R = spatial.assemble_residual(spec.q, grid, bcs, mech, model)
    case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme="CS1",
                       cfl=spec.cfl)
    qg, fg, cg, _, dg = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=1, want_dq=True)
    qw, fw, cw, _, dw = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=2, want_dq=True)
    assert comp_relerr(dw, dg) <= 1e-10
    assert (fw, cw) == (fg, cg)


# ------------------------------------------------------- coupled operator with chemistry


@pytest.mark.parametrize("ns,dims", [(5, (24, 40, 1)), (11, (24, 200, 1)), (16, (20, 70, 1)),
                                     (5, (16, 832, 1))])
def test_ci_chemistry_wavefront_vs_generic_and_oracle(ns, dims):
    """The coupled operator with chemistry on the wavefront (the ns x ns
    species block inverses ride in the CF / CB records and the chain applies
    them, lusgs.py:92-100, 136-144): against the generic hyperplane sweeps of
    the same step, and against the oracle with dOmega injected,
    up to 16 species and at 26 strips."""
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200 import driver, spatial
    from paper_2403_03440_b200.configs import build_case
    spec = C.config3(ns, seed=11, dims=dims, chemistry=True)
    grid, model, bcs, mech = build_case(spec)
    R = spatial.assemble_residual(spec.q, grid, bcs, mech, model)
    case = driver.Case(grid=grid, model=model, bcs=bcs, freestream=None, mech=mech, scheme="CI",
                       cfl=spec.cfl)
    qg, fg, cg, _, dg = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=1, want_dq=True)
    qw, fw, cw, _, dw = driver.implicit_step_raw(case, spec.q, R, spec.cfl, path=2, want_dq=True)
    assert comp_relerr(dw, dg) <= 1e-10
    assert comp_relerr(qw - spec.q, qg - spec.q) <= 1e-10
    assert (fw, cw) == (fg, cg)
    _iteration(spec, ("CI",), chemistry=True, path=2)
