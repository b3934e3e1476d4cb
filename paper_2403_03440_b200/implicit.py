"""Implicit pseudo-time machinery on the GPU (drop-in for reference implicit.py).

Entry points keep the reference's names and signatures:
``local_time_step`` (implicit.py:33-44), ``cell_spectral_radii`` (152-163),
``assemble_lhs`` -> ``ImplicitOperator`` (210-403), ``correct_increment_cs1``
/ ``correct_normalize_cs2`` (113-135).  The operator lives on the device in
the library's compact form (per-cell state + diagonals + face radii); the
reference-shaped fields (w, b, sp_lower, ...) are materialised only when a
caller reads them.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from .device import OP_FIELDS, SCHEMES, SoA, get_engine, is_torch
from .errors import NonPhysicalState, SingularDiagonal
from .mixture import EPS_NEG

MODES = ("CI", "CS1", "CS2")

_UTIL_MODEL = []


def util_engine():
    """Grid-free engine for element-wise utilities (flags + scratch only)."""
    if not _UTIL_MODEL:
        from .configs import cloned_mixture
        _UTIL_MODEL.append(cloned_mixture(1))
    return get_engine(None, _UTIL_MODEL[0])


def _dev(eng, x):
    torch = eng.torch
    if is_torch(x):
        return x.to(device=eng.device, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float))).to(eng.device)


def _out(eng, t, like, shape):
    t = t.reshape(shape)
    if is_torch(like):
        return t.to(like.device)
    a = t.cpu().numpy()
    return a[()] if a.ndim == 0 else a


def local_time_step(lam_inv, lam_vis, lam_S, cfl, J):
    """CFL pseudo-time step dtau = CFL / (J (sum lam_inv + sum lam_vis) + lam_S)."""
    eng = util_engine()
    li = _dev(eng, lam_inv)
    lv = _dev(eng, lam_vis)
    shape = tuple(np.broadcast_shapes(tuple(li.shape[:-1]), tuple(lv.shape[:-1]),
                                      tuple(np.shape(J)), tuple(np.shape(lam_S))))
    n = int(np.prod(shape)) if shape else 1
    li = li.expand(shape + (3,)).contiguous() if tuple(li.shape[:-1]) != shape else li
    lv = lv.expand(shape + (3,)).contiguous() if tuple(lv.shape[:-1]) != shape else lv
    Jt = _dev(eng, J).expand(shape).contiguous() if shape else _dev(eng, J).reshape(1)
    lS_arr = None
    lS_scalar = 0.0
    if np.ndim(lam_S) == 0 and not is_torch(lam_S):
        lS_scalar = float(lam_S)
    else:
        lS_arr = _dev(eng, lam_S).expand(shape).contiguous()
    out = eng.empty(n)
    eng._chk(eng.lib.csb_local_time_step(eng.ctx, n, li.data_ptr(), lv.data_ptr(),
                                         lS_arr.data_ptr() if lS_arr is not None else None,
                                         lS_scalar, float(cfl), Jt.data_ptr(), out.data_ptr(),
                                         ctypes.c_void_p(eng.stream)), "local_time_step")
    eng.check("local_time_step", order=("zero",))
    like = lam_inv if is_torch(lam_inv) else None
    return _out(eng, out, like, shape)


def dual_time_rhs(R, q_m, q_n, q_nm1, theta, dt, volume):
    """RHS = -R - V [(1 + theta)(Q^m - Q^n) - theta (Q^n - Q^{n-1})] / dt
    (implicit.py:47-56) on the device; steady mode (dt None or inf) is -R."""
    if dt is None or not np.isfinite(dt):
        return -R if is_torch(R) else -np.asarray(R)
    from .device import engine_for_ns
    shape = tuple(R.shape)
    nv = shape[-1]
    eng = engine_for_ns(nv - 5)
    n = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
    soa = lambda x: eng.to_soa(_dev(eng, x).reshape(n, nv) if is_torch(x) else
                               np.broadcast_to(np.asarray(x, dtype=float), shape).reshape(n, nv), nv)
    V = _dev(eng, volume).expand(shape[:-1]).contiguous().reshape(n) if len(shape) > 1 else \
        _dev(eng, volume).reshape(1)
    out = eng.empty(nv, n)
    # (named: a temporary's data_ptr() would dangle before the launch)
    tR, tm, tn, tnm1 = soa(R), soa(q_m), soa(q_n), soa(q_nm1)
    eng._chk(eng.lib.csb_dual_time_rhs(eng.ctx, n, V.data_ptr(), tR.data_ptr(), tm.data_ptr(),
                                       tn.data_ptr(), tnm1.data_ptr(), float(theta), float(dt),
                                       out.data_ptr(), ctypes.c_void_p(eng.stream)),
             "dual_time_rhs")
    return eng.from_soa(out, R if is_torch(R) else np.empty(0), shape)


def _q_of(prim, model):
    q = getattr(prim, "_q", None)
    if q is not None:
        return q
    from .mixture import prim_to_cons
    return prim_to_cons(prim, model)


def cell_spectral_radii(prim, grid, model):
    """Unified per-direction radii (lam_inv, lam_vis), each (..., 3), m^3/s."""
    eng = get_engine(grid, model)
    q = _q_of(prim, model)
    qs = eng.to_soa(q, eng.nv)
    li = eng.empty(3, eng.N)
    lv = eng.empty(3, eng.N)
    eng._chk(eng.lib.csb_spectral_radii(eng.ctx, qs.data_ptr(), li.data_ptr(), lv.data_ptr(),
                                        ctypes.c_void_p(eng.stream)), "cell_spectral_radii")
    eng.check("cell_spectral_radii", order=("decode",))
    like = q if is_torch(q) else np.empty(0)
    shp = tuple(eng.dims) + (3,)
    return eng.from_soa(li, like, shp), eng.from_soa(lv, like, shp)


def pseudo_time_step(q, grid, mech, model, cfl, dom_override=None):
    """dtau exactly as _implicit_step computes it (driver.py:235-239):
    cell radii + (chemistry) source radius -> local_time_step, fused on the
    device.  ``dom_override`` injects dOmega (..., ns, ns)."""
    eng = get_engine(grid, model)
    eng.set_mechanism(mech)
    qs = eng.to_soa(q, eng.nv)
    dom = None
    if dom_override is not None and eng.chem_on():
        dom = eng.to_soa(np.asarray(dom_override, float).reshape(tuple(eng.dims) + (eng.ns ** 2,)),
                         eng.ns ** 2)
    out = eng.empty(eng.N)
    eng._chk(eng.lib.csb_time_step(eng.ctx, qs.data_ptr(), float(cfl),
                                   dom.data_ptr() if dom is not None else None, out.data_ptr(),
                                   ctypes.c_void_p(eng.stream)), "time_step")
    eng.check("time_step", order=("decode", "zero"))
    return _out(eng, out, q if is_torch(q) else None, tuple(eng.dims))


class ImplicitOperator:
    """Assembled left-hand side for one pseudo-time step (implicit.py:210-326).

    Device-resident; reference-shaped fields are materialised on access:
    ``w, b, rho, u, lam_face, d_scal, vdom, dinv_species_block, lam_face_sp,
    d_species, sp_lower, sp_upper, sp_scale``.
    """

    def __init__(self, eng, mode, grid, model, qs, dtau_t, offdiag, theta, dt, dom_in, like):
        self._eng = eng
        self.mode = mode
        self.grid = grid
        self.model = model
        self._qs = qs
        self._dtau = dtau_t
        self._offdiag = offdiag
        self._theta = theta
        self._dt = dt
        self._dom_in = dom_in
        self._like = like
        self._gen = None
        self._cache = {}
        self.sp_scale = 0.5 if offdiag == "symmetrized" else 1.0
        self._assemble()

    # -- device ------------------------------------------------------------------
    def _assemble(self):
        eng = self._eng
        dt = -1.0 if self._dt is None or not np.isfinite(self._dt) else float(self._dt)
        eng._chk(eng.lib.csb_assemble(eng.ctx, self._qs.data_ptr(), self._dtau.data_ptr(),
                                      SCHEMES[self.mode], int(self._offdiag == "paper"),
                                      float(self._theta), dt,
                                      self._dom_in.data_ptr() if self._dom_in is not None else None,
                                      ctypes.c_void_p(eng.stream)), "assemble_lhs")
        eng.check("assemble_lhs", order=("decode", "singular"))
        eng._op_gen = getattr(eng, "_op_gen", 0) + 1
        self._gen = eng._op_gen

    def ensure_current(self):
        """Re-assemble if another assemble_lhs on the same grid overwrote the device copy."""
        if getattr(self._eng, "_op_gen", None) != self._gen:
            self._assemble()

    def _field(self, name, comps, shape):
        if name in self._cache:
            return self._cache[name]
        self.ensure_current()
        eng = self._eng
        which = OP_FIELDS[name]
        n = eng.N if name not in ("lam_face0", "lam_face1", "lam_face2", "lam_face_sp0",
                                  "lam_face_sp1", "lam_face_sp2") else None
        if n is None:
            d = int(name[-1])
            fshape = list(eng.dims)
            fshape[d] += 1
            t = eng.empty(int(np.prod(fshape)))
            eng._chk(eng.lib.csb_operator_field(eng.ctx, self._qs.data_ptr(), which, t.data_ptr(),
                                                ctypes.c_void_p(eng.stream)), name)
            out = _out(eng, t, self._like, tuple(fshape))
        else:
            t = eng.empty(comps, eng.N)
            eng._chk(eng.lib.csb_operator_field(eng.ctx, self._qs.data_ptr(), which, t.data_ptr(),
                                                ctypes.c_void_p(eng.stream)), name)
            if comps == 1:
                out = _out(eng, t, self._like, tuple(eng.dims))
            else:
                out = eng.from_soa(t, self._like if self._like is not None else np.empty(0), shape)
        self._cache[name] = out
        return out

    @property
    def nvar(self) -> int:
        return self._eng.nv

    @property
    def w(self):
        return self._field("w", self.nvar, tuple(self._eng.dims) + (self.nvar,))

    @property
    def b(self):
        return self._field("b", self.nvar, tuple(self._eng.dims) + (self.nvar,))

    @property
    def rho(self):
        return self.w[..., 0]

    def _prim(self):
        if "prim" not in self._cache:
            from .mixture import _decode_soa
            self._cache["prim"] = _decode_soa(self._eng, self._qs, self._like)
        return self._cache["prim"]

    @property
    def u(self):
        return self._prim().u

    @property
    def d_scal(self):
        return self._field("d_scal", 1, tuple(self._eng.dims))

    @property
    def lam_face(self):
        return tuple(self._field(f"lam_face{d}", 1, None) for d in range(3))

    @property
    def lam_face_sp(self):
        if self.mode == "CI":
            return None
        return tuple(self._field(f"lam_face_sp{d}", 1, None) for d in range(3))

    @property
    def d_species(self):
        if self.mode == "CI":
            return None
        ns = self._eng.ns
        return self._field("d_species", ns, tuple(self._eng.dims) + (ns,))

    def _sp(self, name):
        if self.mode == "CI":
            return None
        base = self._field(name, 3, tuple(self._eng.dims) + (3,))
        ns = self._eng.ns
        if is_torch(base):
            return base[..., None].expand(base.shape + (ns,)).contiguous()
        return np.repeat(base[..., np.newaxis], ns, axis=-1)

    @property
    def sp_lower(self):
        return self._sp("sp_lower")

    @property
    def sp_upper(self):
        return self._sp("sp_upper")

    @property
    def vdom(self):
        if not self._eng.chem_on() or not (self.mode == "CI" or self._eng.ws_block):
            return None
        ns = self._eng.ns
        t = self._field("vdom", ns * ns, tuple(self._eng.dims) + (ns * ns,))
        return t.reshape(tuple(self._eng.dims) + (ns, ns))

    @property
    def dinv_species_block(self):
        if self.mode != "CI" or not self._eng.chem_on():
            return None
        ns = self._eng.ns
        t = self._field("dinv", ns * ns, tuple(self._eng.dims) + (ns * ns,))
        return t.reshape(tuple(self._eng.dims) + (ns, ns))


def _dtau_device(eng, dtau):
    torch = eng.torch
    if is_torch(dtau):
        t = dtau.to(device=eng.device, dtype=torch.float64)
    else:
        t = torch.as_tensor(np.asarray(dtau, dtype=float), device=eng.device)
    return t.expand(tuple(eng.dims)).contiguous().reshape(eng.N)


def assemble_lhs(q, grid, mode: str, dtau, mech, model, *, theta: float = 0.0,
                 dt: Optional[float] = None, species_offdiag: str = "symmetrized",
                 dom_override=None) -> ImplicitOperator:
    """Build the implicit operator for one iteration (implicit.py:329-403).

    ``dom_override`` (extension): a source Jacobian dOmega
    (..., ns, ns) injected instead of the finite-difference one.
    """
    if mode not in MODES:
        raise ValueError(f"unknown scheme {mode!r}")
    if species_offdiag not in ("symmetrized", "paper"):
        raise ValueError("species_offdiag must be 'symmetrized' or 'paper'")
    eng = get_engine(grid, model)
    eng.set_mechanism(mech)
    if mode == "CI" and eng.chem_on():
        eng.ensure_workspace(True)
    qs = eng.to_soa(q, eng.nv)
    dom = None
    if dom_override is not None and eng.chem_on():
        dom = eng.to_soa(np.asarray(dom_override, float).reshape(tuple(eng.dims) + (eng.ns ** 2,))
                         if not is_torch(dom_override) else
                         dom_override.reshape(tuple(eng.dims) + (eng.ns ** 2,)), eng.ns ** 2)
    like = q if is_torch(q) else None
    return ImplicitOperator(eng, mode, grid, model, qs, _dtau_device(eng, dtau), species_offdiag,
                            theta, dt, dom, like)


def _rows(eng, x, ns):
    return _dev(eng, x).reshape(-1, ns).contiguous()


def _correct(mode, rho_s, d_rho_s, d_rho, eps_neg):
    if eps_neg != EPS_NEG:
        raise ValueError("the device corrections use the reference's eps_neg = 1e-10")
    eng = util_engine()
    rs = np.asarray(rho_s) if not is_torch(rho_s) else rho_s
    ns = rs.shape[-1]
    a = _rows(eng, rho_s, ns)
    b = _rows(eng, d_rho_s, ns)
    rows = a.shape[0]
    c = _dev(eng, d_rho).reshape(-1).expand(rows).contiguous()
    out = eng.empty(rows, ns)
    eng._chk(eng.lib.csb_correct(eng.ctx, mode, rows, ns, a.data_ptr(), b.data_ptr(), c.data_ptr(),
                                 out.data_ptr(), ctypes.c_void_p(eng.stream)), "correct")
    flags, _, _ = eng.status()
    if flags:
        raise NonPhysicalState("consistency correction produced negative species density")
    return _out(eng, out, rho_s if is_torch(rho_s) else None, tuple(rs.shape))


def species_block_inverse(d, V, dOmega):
    """dinv = inv(d I - V dOmega) per cell: the coupled operator's species
    block with chemistry (reference implicit.py:362-368, numpy.linalg.inv),
    on the device as one batched call (csb_batched_inverse: one thread per
    cell up to 23 species, one warp per cell from 24 to 32; in-place
    Gauss-Jordan with partial pivoting).  d, V: (N,);
    dOmega: (N, ns, ns) with ns <= 32.  Raises SingularDiagonal like the
    reference."""
    eng = util_engine()
    torch = eng.torch
    dO = _dev(eng, dOmega)
    if dO.dim() != 3 or dO.shape[1] != dO.shape[2]:
        raise ValueError("dOmega must be (N, ns, ns)")
    N, ns = int(dO.shape[0]), int(dO.shape[1])
    if ns > 32:
        raise ValueError("csb_batched_inverse handles ns <= 32")
    blocks = dO.reshape(N, ns * ns).t().contiguous()
    dd = _dev(eng, d).reshape(N).contiguous()
    vv = _dev(eng, V).reshape(N).contiguous()
    out = torch.empty((ns * ns, N), dtype=torch.float64, device=eng.device)
    fl = torch.zeros(16, dtype=torch.int64, device=eng.device)
    eng._chk(eng.lib.csb_batched_inverse(ns, N, blocks.data_ptr(), dd.data_ptr(), vv.data_ptr(),
                                         out.data_ptr(), fl.data_ptr(), ctypes.c_void_p(eng.stream)),
             "batched_inverse")
    torch.cuda.synchronize()
    if int(fl[0].item()) & (1 << 7):
        raise SingularDiagonal("species diagonal block not invertible")
    res = out.t().reshape(N, ns, ns).contiguous()
    return _out(eng, res, dOmega if is_torch(dOmega) else None, (N, ns, ns))


def correct_increment_cs1(rho_s, d_rho_s, d_rho, eps_neg: float = EPS_NEG):
    """First consistency correction (implicit.py:113-125)."""
    return _correct(1, rho_s, d_rho_s, d_rho, eps_neg)


def correct_normalize_cs2(rho_s, d_rho_s, d_rho, eps_neg: float = EPS_NEG):
    """Second consistency correction (implicit.py:128-135)."""
    return _correct(2, rho_s, d_rho_s, d_rho, eps_neg)


__all__ = ["MODES", "ImplicitOperator", "assemble_lhs", "cell_spectral_radii", "dual_time_rhs",
           "correct_increment_cs1", "correct_normalize_cs2", "local_time_step", "SingularDiagonal",
           "species_block_inverse"]
