"""Generate golden fixtures by running the REAL reference (``/root/reference``).

Run here (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbcache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz``.  Every case stores its own inputs (nodes,
conservative field, species table, BC encoding, reactions) so the tests can
rebuild it without this script.  Outputs are the reference's intermediates of
one implicit iteration, captured stage by stage the way ``_implicit_step``
runs them (reference driver.py:232-251):

  R, P (assemble_residual, return_padded), lam_inv/lam_vis
  (cell_spectral_radii), dOm + lam_S (source_jacobian), dtau
  (local_time_step), every ImplicitOperator field per scheme (assemble_lhs),
  dq* (the numba forward kernel alone), dq (lusgs_solve), q_new (the species
  closure with _check_corrected disabled so inadmissible cells still get
  values), and a per-cell gate mask.

Plus chemistry known-answer vectors and a short steady march history.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import csflow.implicit as ref_implicit  # noqa: E402
import csflow.lusgs as ref_lusgs  # noqa: E402
from csflow.boundary import BoundaryCondition  # noqa: E402
from csflow.chemistry import (Mechanism, Reaction, production_rates, source_jacobian,  # noqa: E402
                              source_spectral_radius)
from csflow.driver import (Case, _implicit_step, _stagnation_monitor, residual_norms,  # noqa: E402
                           steady_solve, unsteady_solve, wall_heat_flux)
from csflow.grid import compute_metrics  # noqa: E402
from csflow.implicit import (assemble_lhs, cell_spectral_radii, dual_time_rhs,  # noqa: E402
                             local_time_step)
from csflow.lusgs import lusgs_solve  # noqa: E402
from csflow.mixture import (MixtureModel, SpeciesData, cons_to_prim, make_primitive,  # noqa: E402
                            prim_to_cons)
from csflow.spatial import assemble_residual  # noqa: E402

from paper_2403_03440_b200 import configs as C  # noqa: E402

KINDS = ("farfield", "supersonic_outflow", "noslip_isothermal", "symmetry", "periodic")
FACES = C.FACES
OUT = {}


def put(case, key, val):
    OUT[f"{case}/{key}"] = np.asarray(val)


def ref_model(spec):
    return MixtureModel(species=tuple(SpeciesData(**vars(s)) for s in spec.species),
                        Pr=spec.Pr, Sc=spec.Sc)


def ref_bcs(spec, model):
    out = {}
    for f in FACES:
        b = spec.bcs[f]
        fs = None
        if b.fs is not None:
            rho, u, T, Y = b.fs
            fs = make_primitive(model, rho=rho, u=u, T=T, Y=Y)
        out[f] = BoundaryCondition(b.kind, freestream=fs, T_wall=b.T_wall, axis=b.axis)
    return out


def ref_mech(spec):
    if not spec.reactions:
        return None
    return Mechanism(reactions=tuple(
        Reaction(np.asarray(r.nu_r, float), np.asarray(r.nu_p, float), r.Af, r.bf, r.Eaf,
                 backward=r.back) for r in spec.reactions))


def store_inputs(name, spec):
    put(name, "nodes", spec.nodes)
    put(name, "q", spec.q)
    put(name, "species", np.array([[s.M, s.cp, s.hf, s.Tref, s.mu_ref, s.T_mu, s.S_mu]
                                   for s in spec.species]))
    put(name, "PrSc", [spec.Pr, spec.Sc])
    put(name, "cfl", spec.cfl)
    ns = spec.ns
    kinds, tw, ax, fs = [], [], [], []
    for f in FACES:
        b = spec.bcs[f]
        kinds.append(KINDS.index(b.kind))
        tw.append(np.nan if b.T_wall is None else b.T_wall)
        ax.append(-1 if b.axis is None else b.axis)
        if b.fs is None:
            fs.append(np.full(5 + ns, np.nan))
        else:
            rho, u, T, Y = b.fs
            fs.append(np.concatenate(([rho], np.asarray(u, float), [T], np.asarray(Y, float))))
    put(name, "bc_kind", kinds)
    put(name, "bc_Twall", tw)
    put(name, "bc_axis", ax)
    put(name, "bc_fs", np.array(fs))
    if spec.reactions:
        put(name, "rx_nu_r", np.array([r.nu_r for r in spec.reactions]))
        put(name, "rx_nu_p", np.array([r.nu_p for r in spec.reactions]))
        put(name, "rx_f", np.array([[r.Af, r.bf, r.Eaf] for r in spec.reactions]))
        put(name, "rx_b", np.array([r.back if r.back is not None else (np.nan,) * 3
                                    for r in spec.reactions]))


def gate_mask(q_new, model, scheme):
    bad = np.zeros(q_new.shape[:3], dtype=bool)
    for idx in np.ndindex(*q_new.shape[:3]):
        try:
            if scheme == "CI":
                if q_new[idx][-1] < -1e-10 * q_new[idx][0]:
                    raise ref_implicit.NonPhysicalState("last species")
            else:
                ref_implicit._check_corrected(q_new[idx][5:], 1e-10)
            cons_to_prim(q_new[idx], model)
        except ref_implicit.NonPhysicalState:
            bad[idx] = True
    return bad


def one_iteration(name, spec, schemes, offdiag="symmetrized", first_order=False):
    store_inputs(name, spec)
    model = ref_model(spec)
    grid = compute_metrics(spec.nodes)
    bcs = ref_bcs(spec, model)
    mech = ref_mech(spec)
    q = spec.q
    put(name, "vol", grid.volume)
    put(name, "Si", grid.Si)
    put(name, "Sj", grid.Sj)
    put(name, "Sk", grid.Sk)
    R, P = assemble_residual(q, grid, bcs, mech, model, first_order=first_order,
                             return_padded=True)
    put(name, "R", R)
    put(name, "P", P)
    walls = [f for f in FACES if spec.bcs[f].kind == "noslip_isothermal"]
    if walls:  # wall heat flux + stagnation monitor (driver.py:132-205)
        qw = wall_heat_flux(P, grid, bcs, model)
        for f in walls:
            put(name, f"qw_{f}", qw[f])
        put(name, "q_stag", _stagnation_monitor(P, grid, bcs, model))
    put(name, "first_order", first_order)
    R1 = assemble_residual(q, grid, bcs, mech, model, first_order=True)
    put(name, "R_first_order", R1)
    prim = cons_to_prim(q, model)
    li, lv = cell_spectral_radii(prim, grid, model)
    put(name, "lam_inv", li)
    put(name, "lam_vis", lv)
    chem_on = mech is not None and mech.enabled and bool(mech.reactions)
    lS = 0.0
    if chem_on:
        dOm = source_jacobian(prim, mech, model)
        put(name, "dOm", dOm)
        put(name, "omega", production_rates(prim, mech, model))
        lS = source_spectral_radius(dOm)
        put(name, "lam_S", lS)
    dtau = local_time_step(li, lv, lS, spec.cfl, grid.J)
    put(name, "dtau", dtau)
    rhs = -R
    for sch in schemes:
        key = f"{sch}" if offdiag == "symmetrized" else f"{sch}_paper"
        op = assemble_lhs(q, grid, sch, dtau, mech, model, species_offdiag=offdiag)
        put(name, f"{key}/w", op.w)
        put(name, f"{key}/b", op.b)
        put(name, f"{key}/d_scal", op.d_scal)
        for d in range(3):
            put(name, f"{key}/lam_face{d}", op.lam_face[d])
        if op.dinv_species_block is not None:
            put(name, f"{key}/dinv", op.dinv_species_block)
        if sch != "CI":
            put(name, f"{key}/d_species", op.d_species)
            put(name, f"{key}/sp_lower", op.sp_lower)
            put(name, f"{key}/sp_upper", op.sp_upper)
            for d in range(3):
                put(name, f"{key}/lam_face_sp{d}", op.lam_face_sp[d])
        # forward sweep alone: dq*
        star = np.zeros_like(rhs)
        lF = op.lam_face
        if sch == "CI":
            has = op.dinv_species_block is not None
            dinv = op.dinv_species_block if has else np.zeros((1, 1, 1, 1, 1))
            ref_lusgs._ci_forward(star, np.ascontiguousarray(rhs), op.w, op.b, op.rho, op.u,
                                  grid.Si, grid.Sj, grid.Sk, lF[0], lF[1], lF[2], op.d_scal,
                                  dinv, has)
        else:
            ref_lusgs._cs_forward(star, np.ascontiguousarray(rhs), op.w, op.b, op.rho, op.u,
                                  grid.Si, grid.Sj, grid.Sk, lF[0], lF[1], lF[2], op.sp_lower,
                                  op.d_scal, 1.0 / op.d_species)
        put(name, f"{key}/dq_star", star)
        dq = lusgs_solve(op, rhs)
        put(name, f"{key}/dq", dq)
        # species closure without the admissibility raise
        saved = ref_implicit._check_corrected
        ref_implicit._check_corrected = lambda *a, **k: None
        try:
            qn = q.copy()
            qn[..., :5] += dq[..., :5]
            if sch == "CI":
                qn[..., 5:] += dq[..., 5:]
                qn[..., -1] = qn[..., 0] - np.sum(qn[..., 5:-1], axis=-1)
            elif sch == "CS1":
                qn[..., 5:] = ref_implicit.correct_increment_cs1(q[..., 5:], dq[..., 5:],
                                                                 dq[..., 0])
            else:
                qn[..., 5:] = ref_implicit.correct_normalize_cs2(q[..., 5:], dq[..., 5:],
                                                                 dq[..., 0])
        finally:
            ref_implicit._check_corrected = saved
        put(name, f"{key}/q_new", qn)
        put(name, f"{key}/gate_bad", gate_mask(qn, model, sch))
    n = residual_norms(R)
    put(name, "norms", [n.flow, n.species, n.density])


def case_chem3d():
    rng = np.random.default_rng(31)
    sp = C.synthetic_species(3, rng)
    dims = (4, 3, 3)
    nodes = C.box_nodes((4e-3, 3e-3, 3e-3), dims)
    rho = rng.uniform(0.5, 1.5, dims) * 1e-2
    vel = rng.uniform(-300.0, 300.0, dims + (3,))
    T = rng.uniform(800.0, 1500.0, dims)
    Y = rng.dirichlet(np.full(3, 5.0), size=dims)
    q = C.encode_state(rho, vel, T, Y, sp)
    Ru = C.R_U
    rx = [C.ReactionSpec(np.array([1.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0]), 3.0e3, 0.5,
                         Ru * 4000.0, back=(2.0e2, 0.0, Ru * 1500.0)),
          C.ReactionSpec(np.array([2.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0]), 5.0e2, -0.3,
                         Ru * 2500.0)]
    fs = (1e-2, (120.0, -30.0, 10.0), 1000.0, np.array([0.3, 0.3, 0.4]))
    bcs = {"imin": C.BCSpec("periodic"), "imax": C.BCSpec("periodic"),
           "jmin": C.BCSpec("noslip_isothermal", T_wall=500.0), "jmax": C.BCSpec("farfield", fs=fs),
           "kmin": C.BCSpec("symmetry"), "kmax": C.BCSpec("supersonic_outflow")}
    return C.CaseSpec("chem3d", nodes, sp, bcs, q, 5.0, reactions=rx)


def case_thin():
    """nj = 1, nk = 2: the degenerate ghost layers in 3-D."""
    rng = np.random.default_rng(41)
    sp = C.air5_species()
    dims = (6, 1, 2)
    nodes = C.box_nodes((6e-3, 1e-3, 2e-3), dims)
    rho = rng.uniform(0.5, 1.5, dims) * 1e-2
    vel = rng.uniform(-400.0, 400.0, dims + (3,))
    T = rng.uniform(500.0, 3000.0, dims)
    Y = rng.dirichlet(np.ones(5), size=dims)
    q = C.encode_state(rho, vel, T, Y, sp)
    fs = (1e-2, (200.0, 0.0, 0.0), 800.0, np.array([0.7, 0.2, 0.05, 0.03, 0.02]))
    bcs = {"imin": C.BCSpec("farfield", fs=fs), "imax": C.BCSpec("supersonic_outflow"),
           "jmin": C.BCSpec("symmetry"), "jmax": C.BCSpec("symmetry", axis=1),
           "kmin": C.BCSpec("periodic"), "kmax": C.BCSpec("periodic")}
    return C.CaseSpec("thin", nodes, sp, bcs, q, 3.0)


def case_warped():
    """Warped 3-D box (non-orthogonal metrics everywhere), wall on kmin."""
    rng = np.random.default_rng(51)
    sp = C.synthetic_species(4, rng)
    dims = (5, 4, 3)
    nodes = C.box_nodes((5e-3, 4e-3, 3e-3), dims)
    nodes[1:-1, 1:-1, 1:-1] += 1.5e-4 * rng.standard_normal(nodes[1:-1, 1:-1, 1:-1].shape)
    rho = rng.uniform(0.5, 1.5, dims) * 1e-2
    vel = rng.uniform(-400.0, 400.0, dims + (3,))
    T = rng.uniform(500.0, 3000.0, dims)
    Y = rng.dirichlet(np.ones(4), size=dims)
    q = C.encode_state(rho, vel, T, Y, sp)
    fs = (1e-2, (300.0, 50.0, -20.0), 900.0, np.array([0.4, 0.3, 0.2, 0.1]))
    bcs = {"imin": C.BCSpec("farfield", fs=fs), "imax": C.BCSpec("supersonic_outflow"),
           "jmin": C.BCSpec("symmetry"), "jmax": C.BCSpec("farfield", fs=fs),
           "kmin": C.BCSpec("noslip_isothermal", T_wall=400.0), "kmax": C.BCSpec("symmetry")}
    return C.CaseSpec("warped", nodes, sp, bcs, q, 8.0)


def chem_rates_case():
    rng = np.random.default_rng(61)
    sp = C.synthetic_species(5, rng)
    rx = C.synthetic_mechanism(5, rng)
    spec = C.CaseSpec("rates", C.box_nodes(1.0, (1, 1, 1)), sp, C.box_bcs(),
                      C.random_state((4, 5, 1), sp, rng), 1.0, reactions=rx)
    store_inputs("rates", spec)
    model = ref_model(spec)
    mech = ref_mech(spec)
    prim = cons_to_prim(spec.q, model)
    put("rates", "omega", production_rates(prim, mech, model))
    dOm = source_jacobian(prim, mech, model)
    put("rates", "dOm", dOm)
    put("rates", "lam_S", source_spectral_radius(dOm))


def march_case():
    """Reference cylinder_case (pkg/tests/test_driver.py:108-123): binary
    mixture, 16x12 O-grid, Mach 2, CFL ramp; 60 steady iterations."""
    a = C.SpeciesSpec("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0)
    b = C.SpeciesSpec("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)
    from csflow.grid import generate_cylinder_ogrid
    nodes = generate_cylinder_ogrid(0.045, 0.25, (16, 12, 1), stretch=1.15)
    sp = [a, b]
    model = MixtureModel(species=(SpeciesData(**vars(a)), SpeciesData(**vars(b))), Pr=0.72, Sc=0.7)
    Y = np.full(2, 0.5)
    chill = make_primitive(model, rho=1.0, T=250.0, Y=Y)
    uinf = 2.0 * float(chill.c)
    inf = make_primitive(model, rho=1.0, T=250.0, u=(uinf, 0.0, 0.0), Y=Y)
    fs = (1.0, (uinf, 0.0, 0.0), 250.0, Y)
    for sch in ("CS1", "CI"):
        spec = C.CaseSpec(f"march_{sch}", nodes, sp, C.cylinder_bcs(fs), None, 20.0)
        grid = compute_metrics(nodes)
        bcs = ref_bcs(spec, model)
        case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, scheme=sch, cfl=20.0,
                    cfl_ramp=(5.0, 2.0, 10), max_iters=60, residual_drop_orders=np.inf,
                    stop_on_absolute_floor=False)
        q0 = case.initial_field()
        spec.q = q0
        store_inputs(spec.name, spec)
        q, hist = steady_solve(case)
        put(spec.name, "res_flow", hist.res_flow)
        put(spec.name, "res_species", hist.res_species)
        put(spec.name, "res_density", hist.res_density)
        put(spec.name, "cfl_used", hist.cfl)
        put(spec.name, "q_stag_hist", hist.q_stag)
        put(spec.name, "q_final", q)
        put(spec.name, "ramp", [5.0, 2.0, 10])


def march_c4_case():
    """Config 4 on a reduced grid (BASELINE.json config 4; the
    history oracle is a reduced grid run through the identical code path):
    48x32 O-grid (geometry as config 2), 11 species, freestream initial
    field, CS1, CFL ramp 1 -> x2 every 8 iterations, 40 iterations."""
    spec = C.config4(dims=(48, 32, 1))
    model = ref_model(spec)
    grid = compute_metrics(spec.nodes)
    bcs = ref_bcs(spec, model)
    rho, u, T, Y = spec.bcs["jmax"].fs
    inf = make_primitive(model, rho=rho, u=u, T=T, Y=Y)
    case = Case(grid=grid, model=model, bcs=bcs, freestream=inf, scheme="CS1", cfl=1000.0,
                cfl_ramp=(1.0, 2.0, 8), max_iters=40, residual_drop_orders=np.inf,
                stop_on_absolute_floor=False)
    spec.q = case.initial_field()
    name = "march_c4"
    store_inputs(name, spec)
    q, hist = steady_solve(case)
    put(name, "res_flow", hist.res_flow)
    put(name, "res_species", hist.res_species)
    put(name, "res_density", hist.res_density)
    put(name, "cfl_used", hist.cfl)
    put(name, "q_final", q)
    put(name, "ramp", [1.0, 2.0, 8])
    put(name, "fs_prim", np.concatenate(([rho], u, [T], Y)))


def generators_case():
    """Reference grid generators (grid.py:102-162) for the device node fill."""
    from csflow.grid import generate_box, generate_cylinder_ogrid
    put("gen", "box", generate_box((0.3, 0.2, 0.1), (7, 5, 3)))
    put("gen", "ogrid", generate_cylinder_ogrid(1.0, 3.5, (20, 16, 2), stretch=1.05))
    put("gen", "ogrid_first_cell", generate_cylinder_ogrid(0.045, 0.145, (8, 16, 1),
                                                           first_cell=1e-4))
    put("gen", "ogrid_quarter", generate_cylinder_ogrid(0.045, 0.2, (12, 9, 1),
                                                        theta_deg=(180.0, 90.0), span=0.02))


def dual_time_case():
    """Dual-time stepping (implicit.py:47-56, 346-348; driver.py:320-359):
    the unsteady right-hand side, one implicit step with the (1+theta)V/dt
    diagonal, and a short unsteady_solve, on a perturbed 3-D box with a
    binary mixture (the reference's box_case idiom, test_driver.py)."""
    rng = np.random.default_rng(71)
    a = C.SpeciesSpec("A", 0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0)
    b = C.SpeciesSpec("B", 0.032, 918.0, 2.5e5, 298.15, 1.919e-5, 273.15, 139.0)
    sp = [a, b]
    dims = (5, 4, 3)
    nodes = C.box_nodes((5e-3, 4e-3, 3e-3), dims)
    Y0 = np.array([0.6, 0.4])
    fs = (1.0, (80.0, -20.0, 10.0), 400.0, Y0)
    bcs_spec = {f: C.BCSpec("farfield", fs=fs) for f in FACES}
    bcs_spec["kmin"] = C.BCSpec("noslip_isothermal", T_wall=350.0)
    rho = 1.0 + 0.05 * rng.standard_normal(dims)
    vel = np.array([80.0, -20.0, 10.0]) + 5.0 * rng.standard_normal(dims + (3,))
    T = 400.0 + 20.0 * rng.standard_normal(dims)
    Yp = np.clip(0.6 + 0.05 * rng.standard_normal(dims), 0.3, 0.9)
    Y = np.stack([Yp, 1.0 - Yp], axis=-1)
    q = C.encode_state(rho, vel, T, Y, sp)
    spec = C.CaseSpec("dual", nodes, sp, bcs_spec, q, 5.0)
    store_inputs("dual", spec)
    model = ref_model(spec)
    grid = compute_metrics(nodes)
    bcs = ref_bcs(spec, model)
    q_n = q * (1.0 + 1e-3 * rng.standard_normal(q.shape))
    q_nm1 = q * (1.0 + 1e-3 * rng.standard_normal(q.shape))
    R = assemble_residual(q, grid, bcs, None, model)
    put("dual", "q_n", q_n)
    put("dual", "q_nm1", q_nm1)
    theta, dt = 2.0, 2e-6
    put("dual", "theta_dt", [theta, dt])
    put("dual", "rhs", dual_time_rhs(R, q, q_n, q_nm1, theta, dt, grid.volume))
    put("dual", "rhs_theta0", dual_time_rhs(R, q, q_n, q_nm1, 0.0, dt, grid.volume))
    fr = make_primitive(model, rho=fs[0], u=fs[1], T=fs[2], Y=fs[3])
    for sch in ("CS1", "CI"):
        case = Case(grid=grid, model=model, bcs=bcs, freestream=fr, scheme=sch, cfl=5.0)
        qn, _ = _implicit_step(case, q, R, 5.0, theta, dt, q_n, q_nm1)
        put("dual", f"{sch}/q_new", qn)
    case = Case(grid=grid, model=model, bcs=bcs, freestream=fr, scheme="CS1", cfl=5.0,
                dt=2e-6, theta=2.0, n_steps=3, inner_max=6, inner_orders=3.0)
    snaps, times, hist = unsteady_solve(case, q0=q)
    put("dual", "snapshots", np.stack(snaps))
    put("dual", "times", times)
    put("dual", "inner_res", hist.res_flow)


def main():
    spec = C.config0(seed=11, dims=(8, 6, 1))
    one_iteration("box_air5", spec, ("CI", "CS1", "CS2"))
    one_iteration("box_air5", spec, ("CI", "CS1"), offdiag="paper")
    spec = C.config2(seed=12, dims=(12, 10, 1), sigma=1.5)
    one_iteration("ogrid_air11", spec, ("CI", "CS1", "CS2"))
    one_iteration("chem3d", case_chem3d(), ("CI", "CS1", "CS2"))
    one_iteration("thin", case_thin(), ("CI", "CS2"), first_order=True)
    one_iteration("warped", case_warped(), ("CI", "CS1"))
    chem_rates_case()
    march_case()
    march_c4_case()
    generators_case()
    dual_time_case()
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **OUT)
    print(f"wrote {path}: {len(OUT)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
