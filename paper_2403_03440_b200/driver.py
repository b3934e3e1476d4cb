"""Steady pseudo-time driver on the GPU (drop-in for reference driver.py).

``Case``, ``GroupedResidual``, ``ConvergenceHistory``, ``residual_norms``,
``_apply_update``, ``_implicit_step``, ``_step_with_retries`` and
``steady_solve`` keep the reference's names, fields and semantics
(driver.py:38-317).  The field stays on the device for the whole march; each
iteration is one residual launch, one norms reduction and one fused implicit
step (csb_implicit_step), with one host sync to read the norms and the device
flag word that drives the CFL-halving retries.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .boundary import FACE_NAMES
from .device import (F_DECODE, F_FACE_T, F_GATE, F_GATE_DECODE, F_KSKIP, F_RES_NONFINITE,
                     SCHEMES, SoA, engine_for_ns, get_engine, is_torch)
from .errors import Diverged, NonPhysicalState, NoWallBoundary
from .mixture import CellPrimitive, prim_to_cons
from .spatial import residual_device

MAX_STEP_RETRIES = 5  # driver.py:35


@dataclass
class Case:
    """Everything one solver run needs (driver.py:38-75)."""

    grid: object
    model: object
    bcs: dict
    freestream: CellPrimitive
    mech: object = None
    scheme: str = "CI"
    cfl: float = 5.0
    cfl_ramp: Optional[tuple] = None
    species_offdiag: str = "symmetrized"
    first_order: bool = False
    max_iters: int = 2000
    residual_drop_orders: float = 6.0
    monitor_every: int = 10
    monitor_window: int = 20
    monitor_rel_change: Optional[float] = None
    dt: Optional[float] = None
    theta: float = 2.0
    n_steps: int = 0
    inner_orders: float = 4.0
    inner_max: int = 60
    stop_on_absolute_floor: bool = True

    def initial_field(self):
        q0 = prim_to_cons(self.freestream, self.model)
        return np.broadcast_to(q0, self.grid.dims + (self.model.nvar,)).copy()

    def cfl_at(self, it: int) -> float:
        if self.cfl_ramp is None:
            return self.cfl
        start, factor, every = self.cfl_ramp
        return min(self.cfl, start * factor ** (it // max(int(every), 1)))


@dataclass
class GroupedResidual:
    flow: float
    species: float
    density: float


@dataclass
class ConvergenceHistory:
    """driver.py:93-125, plus per-iteration retry counts."""

    iters: list = field(default_factory=list)
    res_flow: list = field(default_factory=list)
    res_species: list = field(default_factory=list)
    res_density: list = field(default_factory=list)
    q_stag: list = field(default_factory=list)
    wall_seconds: list = field(default_factory=list)
    implicit_seconds: list = field(default_factory=list)
    cfl: list = field(default_factory=list)
    retries: list = field(default_factory=list)
    metadata: dict = field(default_factory=dict)
    reason: str = ""

    def record(self, it, norms, q_stag, wall_s, imp_s, cfl, retries=0):
        self.iters.append(it)
        self.res_flow.append(norms.flow)
        self.res_species.append(norms.species)
        self.res_density.append(norms.density)
        self.q_stag.append(q_stag)
        self.wall_seconds.append(wall_s)
        self.implicit_seconds.append(imp_s)
        self.cfl.append(cfl)
        self.retries.append(retries)

    def iterations_to_drop(self, orders: float) -> Optional[int]:
        if not self.res_density:
            return None
        target = self.res_density[0] * 10.0 ** (-orders)
        for it, r in zip(self.iters, self.res_density):
            if r <= target:
                return it
        return None


def _norms_device(eng, R_t, out=None):
    out = eng.empty(4) if out is None else out
    eng._chk(eng.lib.csb_residual_norms(eng.ctx, R_t.shape[1], R_t.data_ptr(), out.data_ptr(),
                                        ctypes.c_void_p(eng.stream)), "residual_norms")
    return out


def residual_norms(R) -> GroupedResidual:
    """Grouped L2 norms (driver.py:85-90) as one device reduction."""
    if isinstance(R, SoA):
        t = R.t
        eng = engine_for_ns(t.shape[0] - 5)
    else:
        nv = int(np.shape(R)[-1])
        eng = engine_for_ns(nv - 5)
        t = eng.to_soa(R, nv)
    v = _norms_device(eng, t).cpu().numpy()
    return GroupedResidual(flow=float(v[0]), species=float(v[1]), density=float(v[2]))


def _apply_update(q, dq, scheme, model):
    """Species closure (driver.py:216-229) on the device; raises like the
    reference when the correction / last-species reconstruction goes negative."""
    eng = get_engine(None, model)
    qa = q if (is_torch(q) or isinstance(q, SoA)) else np.asarray(q, dtype=float)
    shape = tuple(qa.shape if not isinstance(qa, SoA) else qa.dims + (model.nvar,))
    n = int(np.prod(shape[:-1]))
    qs = eng.to_soa(qa.reshape(n, model.nvar) if not isinstance(qa, SoA) else qa, model.nvar)
    dqa = dq if (is_torch(dq) or isinstance(dq, SoA)) else np.asarray(dq, dtype=float)
    ds = eng.to_soa(dqa.reshape(n, model.nvar) if not isinstance(dqa, SoA) else dqa, model.nvar)
    qn = eng.empty(model.nvar, n)
    eng._chk(eng.lib.csb_apply_update(eng.ctx, n, qs.data_ptr(), ds.data_ptr(), SCHEMES[scheme],
                                      qn.data_ptr(), ctypes.c_void_p(eng.stream)), "_apply_update")
    flags, cell, _ = eng.status()
    if flags & F_GATE:
        raise NonPhysicalState("consistency correction produced negative species density"
                               if scheme != "CI" else "reconstructed last species went negative")
    if isinstance(q, SoA):
        return SoA(qn, q.dims)
    return eng.from_soa(qn, q, shape)


# --------------------------------------------------------------------------
# wall heat flux monitor (driver.py:132-205)
# --------------------------------------------------------------------------

def _wall_faces(bcs):
    return [name for name in FACE_NAMES if bcs[name].kind == "noslip_isothermal"]


class _WallGeom:
    """Per wall face: the three node planes nearest the wall (plane 0 = the
    wall) uploaded once, the input csb_wall_heat_flux reads its geometry from
    (face normal, face and cell centroids, wall distances)."""

    def __init__(self, eng, grid, bcs):
        nodes = np.asarray(grid.nodes, dtype=float)
        self.faces = {}
        for name in _wall_faces(bcs):
            fid = FACE_NAMES.index(name)
            axis, side = divmod(fid, 2)
            n = eng.dims[axis]
            planes = [n, n - 1, n - 2] if side else [0, 1, 2]
            slab = np.ascontiguousarray(np.moveaxis(nodes, axis, 0)[planes])
            shape = tuple(d for a, d in enumerate(eng.dims) if a != axis)
            self.faces[name] = (fid, shape, eng.torch.from_numpy(slab).to(eng.device))


def _wall_flux_device(eng, q_soa, geom):
    """{face: (qw, p1)} device tensors shaped like the wall (driver.py:132-184)."""
    out = {}
    for name, (fid, shape, slab) in geom.faces.items():
        qw = eng.empty(*shape)
        pw = eng.empty(*shape)
        eng._chk(eng.lib.csb_wall_heat_flux(eng.ctx, fid, q_soa.data_ptr(), slab.data_ptr(),
                                            qw.data_ptr(), pw.data_ptr(),
                                            ctypes.c_void_p(eng.stream)), "wall_heat_flux")
        out[name] = (qw, pw)
    return out


def wall_heat_flux(P_or_q, grid, bcs, model):
    """Wall-normal heat flux (W/m^2, positive into the wall) per wall face
    (driver.py:132-184), computed on the device.  Accepts the padded
    primitive array P of the reference (ni+4, nj+4, nk+4, 6+ns) or the
    conservative field (any flavour)."""
    if not _wall_faces(bcs):
        raise NoWallBoundary("no noslip_isothermal boundary in this case")
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    arr = P_or_q
    if not isinstance(arr, SoA) and tuple(np.shape(arr)[:3]) == tuple(n + 4 for n in grid.dims):
        # interior of P -> conservative (rho, u, T, Y of the padded layout)
        a = arr[2:-2, 2:-2, 2:-2]
        ns = eng.ns
        prim = CellPrimitive(rho=a[..., 0], u=a[..., 1:4], p=a[..., 4], T=a[..., 5 + ns],
                             Y=a[..., 5:5 + ns], c=None, gamma=None, h=None, Ek=None)
        arr = prim_to_cons(prim, model)
    qs = eng.to_soa(arr, eng.nv)
    res = _wall_flux_device(eng, qs, _WallGeom(eng, grid, bcs))
    eng.check("wall_heat_flux", order=("decode",))
    like = P_or_q if is_torch(P_or_q) else None
    return {k: (v[0] if like is not None else v[0].cpu().numpy()) for k, v in res.items()}


def _stagnation_monitor_device(eng, q_soa, geom):
    """Heat flux at the wall cell holding the peak wall pressure
    (driver.py:187-205): per face a device argmax over p1, then the first
    face with the strictly largest peak."""
    if not geom.faces:
        return float("nan")
    picks = []
    for name, (qw, pw) in _wall_flux_device(eng, q_soa, geom).items():
        o = eng.empty(3)
        eng._chk(eng.lib.csb_argmax_pick(pw.numel(), pw.data_ptr(), qw.data_ptr(), o.data_ptr(),
                                         ctypes.c_void_p(eng.stream)), "stagnation monitor")
        picks.append(o)
    vals = eng.torch.stack(picks).cpu().numpy()
    best, best_p = float("nan"), -np.inf
    for pmax, qv, _ in vals:
        if pmax > best_p:
            best_p, best = float(pmax), float(qv)
    return best


# --------------------------------------------------------------------------
# implicit step and the steady march
# --------------------------------------------------------------------------

class _Stepper:
    """Device buffers of one march."""

    def __init__(self, case):
        self.case = case
        self.eng = eng = get_engine(case.grid, case.model)
        eng.set_bcs(case.bcs)
        eng.set_mechanism(case.mech)
        if case.scheme == "CI" and eng.chem_on():
            eng.ensure_workspace(True)
        self.scheme = SCHEMES[case.scheme]
        self.paper = int(case.species_offdiag == "paper")
        self.R = eng.empty(eng.nv, eng.N)
        self.norms = eng.empty(4)
        torch = eng.torch
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)

    def implicit(self, q_t, R_t, cfl, out_t):
        """One fused implicit step; returns (ok, flags, seconds)."""
        eng = self.eng
        self.ev0.record()
        eng._chk(eng.lib.csb_implicit_step(eng.ctx, q_t.data_ptr(), R_t.data_ptr(), float(cfl),
                                           self.scheme, self.paper, None, out_t.data_ptr(),
                                           ctypes.c_void_p(eng.stream)), "_implicit_step")
        self.ev1.record()
        flags, cell, cnt = eng.status()
        secs = self.ev0.elapsed_time(self.ev1) * 1e-3
        return flags, cell, secs

    def implicit_dual(self, q_t, rhs_t, cfl, theta, dt, out_t):
        """One dual-time implicit step from a formed rhs; (flags, cell, seconds)."""
        eng = self.eng
        self.ev0.record()
        eng._chk(eng.lib.csb_implicit_step_rhs(eng.ctx, q_t.data_ptr(), rhs_t.data_ptr(), float(cfl),
                                               self.scheme, self.paper, float(theta), float(dt),
                                               out_t.data_ptr(), ctypes.c_void_p(eng.stream)),
                 "_implicit_step")
        self.ev1.record()
        flags, cell, cnt = eng.status()
        return flags, cell, self.ev0.elapsed_time(self.ev1) * 1e-3

    def dual_rhs(self, R_t, qm_t, qn_t, qnm1_t, theta, dt, out_t):
        eng = self.eng
        eng._chk(eng.lib.csb_dual_time_rhs(eng.ctx, eng.N, eng.vol.data_ptr(), R_t.data_ptr(),
                                           qm_t.data_ptr(), qn_t.data_ptr(), qnm1_t.data_ptr(),
                                           float(theta), float(dt), out_t.data_ptr(),
                                           ctypes.c_void_p(eng.stream)), "dual_time_rhs")
        return out_t


def _is_dual(dt):
    if dt is None or not np.isfinite(dt):
        return False
    if dt <= 0.0:
        raise ValueError(f"physical time step must be positive, got {dt!r}")
    return True


def _implicit_step(case, q, R, cfl, theta=0.0, dt=None, q_n=None, q_nm1=None):
    """One LU-SGS update at fixed CFL; returns (q_new, implicit_seconds)
    (driver.py:232-251).  With a physical dt the right-hand side is the
    dual-time one and (1 + theta) V / dt joins the diagonal."""
    st = _Stepper(case)
    eng = st.eng
    qs = eng.to_soa(q, eng.nv)
    Rs = eng.to_soa(R, eng.nv)
    out = eng.empty(eng.nv, eng.N)
    if _is_dual(dt):
        rhs = st.dual_rhs(Rs, qs, eng.to_soa(q_n, eng.nv), eng.to_soa(q_nm1, eng.nv), theta, dt,
                          eng.empty(eng.nv, eng.N))
        flags, cell, secs = st.implicit_dual(qs, rhs, cfl, theta, dt, out)
    else:
        flags, cell, secs = st.implicit(qs, Rs, cfl, out)
    flags &= ~F_KSKIP
    if flags:
        eng.raise_for(flags, cell, "_implicit_step")
    if isinstance(q, SoA):
        return SoA(out, eng.dims), secs
    return eng.from_soa(out, q, tuple(eng.dims) + (eng.nv,)), secs


def implicit_step_raw(case, q, R, cfl, dom_override=None, path=0, want_dq=False):
    """Fused implicit step that reports instead of raising:
    returns (q_new, flags, gate_count, first_bad_cell) [+ dq].
    ``dom_override`` injects dOmega (..., ns, ns); ``path``: 0
    auto, 1 generic hyperplane sweeps, 2 the 2-D wavefront path."""
    st = _Stepper(case)
    eng = st.eng
    qs = eng.to_soa(q, eng.nv)
    Rs = eng.to_soa(R, eng.nv)
    dom = None
    if dom_override is not None:
        dom = eng.to_soa(np.asarray(dom_override, float).reshape(tuple(eng.dims) + (eng.ns ** 2,)),
                         eng.ns ** 2)
    out = eng.empty(eng.nv, eng.N)
    dqo = eng.empty(eng.nv, eng.N) if want_dq else None
    eng._chk(eng.lib.csb_implicit_step_ex(eng.ctx, qs.data_ptr(), Rs.data_ptr(), float(cfl),
                                          st.scheme, st.paper,
                                          dom.data_ptr() if dom is not None else None,
                                          out.data_ptr(), dqo.data_ptr() if dqo is not None else None,
                                          int(path), ctypes.c_void_p(eng.stream)),
             "_implicit_step")
    flags, cell, cnt = eng.status()
    like = q if is_torch(q) else np.empty(0)
    shape = tuple(eng.dims) + (eng.nv,)
    res = (eng.from_soa(out, like, shape), flags & ~F_KSKIP, cnt, cell)
    if want_dq:
        res = res + (eng.from_soa(dqo, like, shape),)
    return res


def _step_device(st, q_t, R_t, cfl, out_t, dual=None):
    """_step_with_retries (driver.py:254-263) on device buffers; ``dual`` =
    (rhs, theta, dt) runs dual-time steps from the formed rhs.
    Returns (cfl_used, implicit_seconds, retries)."""
    eng = st.eng
    total = 0.0
    for attempt in range(MAX_STEP_RETRIES + 1):
        if dual is None:
            flags, cell, secs = st.implicit(q_t, R_t, cfl, out_t)
        else:
            flags, cell, secs = st.implicit_dual(q_t, dual[0], cfl, dual[1], dual[2], out_t)
        total += secs
        flags &= ~F_KSKIP
        # first failure in the reference's stage order (driver.py:235-250):
        # decode (NonPhysicalState, retried) -> dtau (ZeroWavespeed) ->
        # assembly/sweeps (SingularDiagonal) -> closure + gate (retried)
        if flags & F_DECODE:
            nonphys = True
        else:
            eng.raise_for(flags, cell, "_implicit_step", order=("zero", "singular"))
            nonphys = bool(flags & (F_GATE | F_GATE_DECODE))
        if not nonphys:
            return cfl, total, attempt
        if attempt == MAX_STEP_RETRIES:
            raise Diverged(f"step failed after {MAX_STEP_RETRIES} CFL halvings (CFL={cfl:g})")
        cfl *= 0.5
    raise AssertionError("unreachable")


def _reference_density_residual(case) -> float:
    """driver.py:208-213."""
    inf = case.freestream
    speed = float(np.linalg.norm(inf.u) + inf.c)
    areas = [np.linalg.norm(case.grid.face_areas(d), axis=-1).mean() for d in range(3)]
    return float(inf.rho) * speed * max(areas) * np.sqrt(case.grid.ncells)


def steady_solve(case, q0=None, *, return_device=False, device_march=True):
    """March to steady state; returns (q, ConvergenceHistory) (driver.py:266-317).

    The loop runs on the device (csb_march_*): one CUDA graph per chunk of
    iterations takes every decision of the reference's loop -- residual
    norms, NaN check, absolute-floor / residual-drop / monitor-plateau stops,
    the ramped CFL times cfl_scale, the CFL-halving retries of each implicit
    step and the x1.2 recovery -- so the host reads the history once per
    chunk.  Chunks end where the stagnation heat-flux monitor samples the
    state (every ``monitor_every`` iterations and at iteration 1), which the
    host evaluates on the device between chunks and turns into the plateau
    decision.  ``device_march=False`` runs the host-driven loop."""
    if not device_march:
        return _steady_solve_host(case, q0, return_device=return_device)
    from ._lib import MarchParams
    st = _Stepper(case)
    eng = st.eng
    torch = eng.torch
    nv, N = eng.nv, eng.N
    q_init = case.initial_field() if q0 is None else q0
    q = eng.to_soa(q_init, nv).clone()
    q_alt = eng.empty(nv, N)
    rows = max(int(case.max_iters), 1)
    hist_dev = eng.zeros(rows, 6)
    cfl_tab = torch.tensor([case.cfl_at(i) for i in range(rows)], dtype=torch.float64,
                           device=eng.device)
    orders = case.residual_drop_orders
    params = MarchParams(st.scheme, st.paper, int(bool(case.first_order)), MAX_STEP_RETRIES,
                         1e-12 * _reference_density_residual(case) if case.stop_on_absolute_floor
                         else -1.0,
                         10.0 ** (-orders) if np.isfinite(orders) else -1.0)
    stream = ctypes.c_void_p(eng.stream)
    eng._chk(eng.lib.csb_march_begin(eng.ctx, ctypes.byref(params), q.data_ptr(),
                                     q_alt.data_ptr(), hist_dev.data_ptr(), rows,
                                     cfl_tab.data_ptr(), stream), "steady_solve")
    hist = ConvergenceHistory(metadata={
        "scheme": case.scheme, "cfl": case.cfl, "cfl_ramp": case.cfl_ramp,
        "monitor_every": case.monitor_every, "monitor_window": case.monitor_window,
        "device_march": True,
    })
    walls = bool(_wall_faces(case.bcs))
    geom = _WallGeom(eng, case.grid, case.bcs) if walls else None
    monitoring = case.monitor_rel_change is not None or walls
    every = max(int(case.monitor_every), 1)
    samples, sample_at = [], {}
    ints = (ctypes.c_int * 4)()
    reals = (ctypes.c_double * 4)()
    done, clear = 0, 0
    try:
        while done < case.max_iters:
            it_next = done + 1
            plateau_at = 0
            if monitoring and (it_next % every == 0 or it_next == 1):
                sample = _stagnation_monitor_device(eng, q, geom) if walls else float("nan")
                samples.append(sample)
                sample_at[it_next] = sample
                if case.monitor_rel_change is not None and len(samples) >= case.monitor_window:
                    w = np.array(samples[-case.monitor_window:])
                    if np.all(np.isfinite(w)) and np.max(np.abs(w - w[-1])) \
                            <= case.monitor_rel_change * max(abs(w[-1]), 1e-300):
                        plateau_at = it_next
            it_last = (it_next // every + 1) * every - 1 if monitoring else case.max_iters
            it_last = min(max(it_last, it_next), case.max_iters)
            t0 = time.perf_counter()
            eng._chk(eng.lib.csb_march_run(eng.ctx, it_last, plateau_at, clear, stream),
                     "steady_solve")
            eng._chk(eng.lib.csb_march_state(eng.ctx, ints, reals, stream), "steady_solve")
            wall = time.perf_counter() - t0
            it_now, stop, parity = ints[0], ints[1], ints[2]
            if it_now > done:
                rows_new = hist_dev[done:it_now].cpu().numpy()
                per = wall / (it_now - done)
                for k, row in enumerate(rows_new):
                    it = done + 1 + k
                    hist.record(it, GroupedResidual(float(row[0]), float(row[1]), float(row[2])),
                                sample_at.get(it, float("nan")), per,
                                per if row[5] == 0 else 0.0, float(row[3]), int(row[4]))
            done = it_now
            clear = 0
            if parity:
                q.copy_(q_alt)
                clear = 1
            if stop:
                _march_stop(eng, stop, done, reals, hist)
                break
        else:
            hist.reason = "max_iters"
    finally:
        eng.lib.csb_march_end(eng.ctx)
    if return_device:
        return SoA(q, eng.dims), hist
    like = q0 if (q0 is not None and is_torch(q0)) else np.empty(0)
    return eng.from_soa(q, like, tuple(eng.dims) + (eng.nv,)), hist


_MARCH_REASONS = {1: "converged_absolute", 2: "converged_residual_drop",
                  3: "converged_monitor_plateau"}


def _march_stop(eng, stop, done, reals, hist):
    """Map a device stop code onto the reference's outcome (driver.py:266-317)."""
    if stop in _MARCH_REASONS:
        hist.reason = _MARCH_REASONS[stop]
        return
    if stop == 4:
        raise Diverged(f"non-finite residual norm at iteration {done + 1}")
    if stop == 5:
        raise Diverged(f"step failed after {MAX_STEP_RETRIES} CFL halvings (CFL={reals[1]:g})")
    flags, cell, _ = eng.status()
    flags &= ~F_KSKIP
    if stop == 8:
        eng.raise_for(flags, cell, "assemble_residual", order=("decode",))
        raise NonPhysicalState("assemble_residual: non-physical state")
    eng.raise_for(flags, cell, "_implicit_step", order=("zero", "singular"))
    raise Diverged(f"march stopped (code {stop})")


def _steady_solve_host(case, q0=None, *, return_device=False):
    """steady_solve with the loop on the host: one residual + norms read and
    one fused implicit step (+ flag read) per iteration.  Kept as the A/B
    reference of the device march."""
    st = _Stepper(case)
    eng = st.eng
    q_init = case.initial_field() if q0 is None else q0
    q = eng.to_soa(q_init, eng.nv).clone()
    q_next = eng.empty(eng.nv, eng.N)
    hist = ConvergenceHistory(metadata={
        "scheme": case.scheme, "cfl": case.cfl, "cfl_ramp": case.cfl_ramp,
        "monitor_every": case.monitor_every, "monitor_window": case.monitor_window,
    })
    ref_floor = 1e-12 * _reference_density_residual(case)
    cfl_scale = 1.0
    samples = []
    walls = bool(_wall_faces(case.bcs))
    geom = _WallGeom(eng, case.grid, case.bcs) if walls else None
    for it in range(1, case.max_iters + 1):
        t0 = time.perf_counter()
        residual_device(eng, q, case.first_order, R=st.R)
        v = _norms_device(eng, st.R, st.norms).cpu().numpy()
        norms = GroupedResidual(float(v[0]), float(v[1]), float(v[2]))
        if not np.isfinite(norms.flow) or not np.isfinite(norms.species):
            raise Diverged(f"non-finite residual norm at iteration {it}")
        sample = float("nan")
        if case.monitor_rel_change is not None or walls:
            if it % case.monitor_every == 0 or it == 1:
                sample = _stagnation_monitor_device(eng, q, geom) if walls else float("nan")
                samples.append(sample)
        cfl_now = case.cfl_at(it - 1) * cfl_scale
        if case.stop_on_absolute_floor and norms.density <= ref_floor:
            hist.record(it, norms, sample, time.perf_counter() - t0, 0.0, cfl_now)
            hist.reason = "converged_absolute"
            break
        drop = (hist.res_density[0] * 10.0 ** (-case.residual_drop_orders)
                if hist.res_density and np.isfinite(case.residual_drop_orders) else None)
        if drop is not None and norms.density <= drop:
            hist.record(it, norms, sample, time.perf_counter() - t0, 0.0, cfl_now)
            hist.reason = "converged_residual_drop"
            break
        if case.monitor_rel_change is not None and len(samples) >= case.monitor_window:
            w = np.array(samples[-case.monitor_window:])
            if np.all(np.isfinite(w)) and np.max(np.abs(w - w[-1])) \
                    <= case.monitor_rel_change * max(abs(w[-1]), 1e-300):
                hist.record(it, norms, sample, time.perf_counter() - t0, 0.0, cfl_now)
                hist.reason = "converged_monitor_plateau"
                break
        cfl_used, t_imp, retries = _step_device(st, q, st.R, cfl_now, q_next)
        q, q_next = q_next, q
        if cfl_used < cfl_now:
            cfl_scale *= cfl_used / cfl_now
        else:
            cfl_scale = min(1.0, cfl_scale * 1.2)
        hist.record(it, norms, sample, time.perf_counter() - t0, t_imp, cfl_used, retries)
    else:
        hist.reason = "max_iters"
    if return_device:
        return SoA(q, eng.dims), hist
    like = q0 if (q0 is not None and is_torch(q0)) else np.empty(0)
    return eng.from_soa(q, like, tuple(eng.dims) + (eng.nv,)), hist


def _step_with_retries(case, q, R, cfl, theta=0.0, dt=None, q_n=None, q_nm1=None):
    """Implicit step with CFL halving on NonPhysicalState (driver.py:254-263);
    returns ((q_new, implicit_seconds), cfl_used)."""
    st = _Stepper(case)
    eng = st.eng
    qs, Rs = eng.to_soa(q, eng.nv), eng.to_soa(R, eng.nv)
    out = eng.empty(eng.nv, eng.N)
    dual = None
    if _is_dual(dt):
        dual = (st.dual_rhs(Rs, qs, eng.to_soa(q_n, eng.nv), eng.to_soa(q_nm1, eng.nv), theta, dt,
                            eng.empty(eng.nv, eng.N)), theta, dt)
    cfl_used, secs, _ = _step_device(st, qs, Rs, cfl, out, dual)
    if isinstance(q, SoA):
        return (SoA(out, eng.dims), secs), cfl_used
    return (eng.from_soa(out, q, tuple(eng.dims) + (eng.nv,)), secs), cfl_used


def unsteady_solve(case, q0=None):
    """Dual-time unsteady march; returns (snapshots, times, ConvergenceHistory)
    (driver.py:320-359).  Physical step 1 runs first order in time
    (theta = 0); each physical step iterates in pseudo time until the inner
    residual |rhs| has dropped ``inner_orders`` decades or ``inner_max``
    iterations ran.  Everything stays on the device; one small read per inner
    iteration (the rhs norm) drives the stopping test."""
    if case.dt is None or not np.isfinite(case.dt) or case.dt <= 0:
        raise ValueError("unsteady_solve requires a positive physical dt")
    st = _Stepper(case)
    eng = st.eng
    nv, N = eng.nv, eng.N
    q_init = case.initial_field() if q0 is None else q0
    q_n = eng.to_soa(q_init, nv).clone()
    q_nm1 = q_n.clone()
    like = q0 if (q0 is not None and is_torch(q0)) else np.empty(0)
    shape = tuple(eng.dims) + (nv,)
    snap = lambda t: eng.from_soa(t, like, shape)
    snapshots, times = [snap(q_n)], [0.0]
    hist = ConvergenceHistory(metadata={"scheme": case.scheme, "dt": case.dt, "theta": case.theta})
    rhs = eng.empty(nv, N)
    q_next = eng.empty(nv, N)
    ss = eng.empty(1)
    for step in range(1, case.n_steps + 1):
        theta = 0.0 if step == 1 else case.theta
        q_m = q_n.clone()
        inner0 = None
        for _inner in range(1, case.inner_max + 1):
            t0 = time.perf_counter()
            residual_device(eng, q_m, case.first_order, R=st.R)
            st.dual_rhs(st.R, q_m, q_n, q_nm1, theta, case.dt, rhs)
            eng._chk(eng.lib.csb_sum_squares(eng.ctx, nv * N, rhs.data_ptr(), ss.data_ptr(),
                                             ctypes.c_void_p(eng.stream)), "inner residual")
            rnorm = float(np.sqrt(ss.item()))
            if inner0 is None:
                inner0 = max(rnorm, 1e-300)
            if not np.isfinite(rnorm):
                raise Diverged(f"non-finite inner residual at step {step}")
            if rnorm <= inner0 * 10.0 ** (-case.inner_orders) or rnorm == 0.0:
                break
            _, t_imp, _ = _step_device(st, q_m, st.R, case.cfl, q_next, (rhs, theta, case.dt))
            q_m, q_next = q_next, q_m
            hist.record(len(hist.iters) + 1, GroupedResidual(rnorm, rnorm, rnorm), float("nan"),
                        time.perf_counter() - t0, t_imp, case.cfl)
        q_nm1, q_n = q_n, q_m
        snapshots.append(snap(q_n))
        times.append(step * case.dt)
    return snapshots, times, hist


__all__ = ["Case", "ConvergenceHistory", "GroupedResidual", "MAX_STEP_RETRIES", "residual_norms",
           "steady_solve", "unsteady_solve", "wall_heat_flux", "_apply_update", "_implicit_step",
           "_step_with_retries"]
