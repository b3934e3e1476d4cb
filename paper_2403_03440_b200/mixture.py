"""Mixture description and state conversion, on the device.

Schema: a mixture is an ordered set of constant-cp species with Sutherland
viscosity plus Prandtl and Schmidt numbers (the fields of reference
mixture.py:33-104).  The solver reads any object with that shape -- the
reference's own ``MixtureModel`` included -- through ``species_table``; the
classes below are a minimal stand-alone implementation of it.

The conversions run in the sm_100a library: ``cons_to_prim``
(mixture.py:287-307, clipping and renormalisation included) through
``csb_cons_to_prim``; ``make_primitive`` and ``prim_to_cons``
(mixture.py:310-351) through ``csb_primitive``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .errors import NonPhysicalState

R_UNIVERSAL = 8.314462618  # J/(mol K), mixture.py:26
EPS_NEG = 1e-10            # mixture.py:30
SPECIES_FIELDS = ("M", "cp", "hf", "Tref", "mu_ref", "T_mu", "S_mu")


class SpeciesData(NamedTuple):
    """One species record: molar mass [kg/mol], cp [J/(kg K)], heat of
    formation [J/kg] at Tref [K], Sutherland (mu_ref, T_mu, S_mu)."""

    name: str
    M: float
    cp: float
    hf: float
    Tref: float
    mu_ref: float
    T_mu: float
    S_mu: float


def species_table(model):
    """Per-species float64 columns of any mixture-shaped object (``.species``
    records with the SPECIES_FIELDS attributes), in the order the C ABI's
    csb_set_model expects."""
    cols = {k: np.ascontiguousarray([float(getattr(sp, k)) for sp in model.species], dtype=float)
            for k in SPECIES_FIELDS}
    return cols


def _validate(names, tab, Pr, Sc):
    problems = []
    if not names:
        problems.append("a mixture needs at least one species")
    if len(set(names)) != len(names):
        problems.append("species names repeat")
    for name, M, cp, mu in zip(names, tab["M"], tab["cp"], tab["mu_ref"]):
        if not M > 0.0:
            problems.append(f"{name}: molar mass {M!r} is not positive")
        elif not cp > R_UNIVERSAL / M:
            problems.append(f"{name}: cp {cp!r} leaves cv = cp - R_u/M <= 0")
        if mu < 0.0:
            problems.append(f"{name}: mu_ref {mu!r} is negative")
    if not (Pr > 0.0 and Sc > 0.0):
        problems.append(f"Pr and Sc must be > 0 (got {Pr!r}, {Sc!r})")
    if problems:
        raise ValueError("; ".join(problems))


class MixtureModel:
    """Ordered species + Pr, Sc; derived per-species arrays M, cp_s, hf_s,
    Tref_s, R_s = R_u / M and b_s = hf - cp Tref."""

    def __init__(self, species, Pr=0.72, Sc=0.7):
        self.species = tuple(species)
        self.Pr = float(Pr)
        self.Sc = float(Sc)
        tab = species_table(self)
        _validate([sp.name for sp in self.species], tab, self.Pr, self.Sc)
        self.M, self.cp_s, self.hf_s, self.Tref_s = tab["M"], tab["cp"], tab["hf"], tab["Tref"]
        self.R_s = R_UNIVERSAL / self.M
        self.b_s = self.hf_s - self.cp_s * self.Tref_s

    @property
    def ns(self) -> int:
        return len(self.species)

    @property
    def nvar(self) -> int:
        return 5 + len(self.species)

    def species_index(self, name: str) -> int:
        names = [sp.name for sp in self.species]
        if name not in names:
            raise KeyError(f"unknown species {name!r}")
        return names.index(name)

    def table(self):
        return species_table(self)


@dataclass(frozen=True)
class CellPrimitive:
    """Decoded primitive state (fields of reference mixture.py:216-232)."""

    rho: object
    u: object
    p: object
    T: object
    Y: object
    c: object
    gamma: object
    h: object
    Ek: object


class DevicePrimitive(CellPrimitive):
    """CellPrimitive produced on the device; keeps the conservative field so
    downstream device calls (cell_spectral_radii, ...) need not re-encode."""


def padded_vector(prim: CellPrimitive, ns: int):
    """[rho, u, v, w, p, Y.., T] of a single state (fields.py:31-36 layout)."""
    parts = (prim.rho, prim.u, prim.p, prim.Y, prim.T)
    sizes = (1, 3, 1, ns, 1)
    return np.concatenate([np.asarray(x, dtype=float).reshape(n) for x, n in zip(parts, sizes)])


def _prim_from_raw(out, shape, ns, like):
    """csb_cons_to_prim / csb_primitive layout (12 + ns, n) -> CellPrimitive."""
    from .device import is_torch
    if is_torch(like):
        o = out.to(like.device)
        f = lambda k: o[k].reshape(shape)
        Y = o[12:].T.reshape(shape + (ns,))
        u = o[1:4].T.reshape(shape + (3,))
    else:
        o = out.cpu().numpy()
        f = lambda k: o[k].reshape(shape)
        Y = np.ascontiguousarray(o[12:].T.reshape(shape + (ns,)))
        u = np.ascontiguousarray(o[1:4].T.reshape(shape + (3,)))
    return DevicePrimitive(rho=f(0), u=u, p=f(4), T=f(5), Y=Y, c=f(6), gamma=f(7), h=f(8),
                           Ek=f(9))


def _decode_soa(eng, qs, like, n=None):
    """Device decode of SoA q (nv, N) -> CellPrimitive shaped like the grid."""
    n = eng.N if n is None else n
    out = eng.empty(12 + eng.ns, n)
    eng._chk(eng.lib.csb_cons_to_prim(eng.ctx, n, qs.data_ptr(), out.data_ptr(),
                                      ctypes.c_void_p(eng.stream)), "cons_to_prim")
    eng.check("cons_to_prim", order=("decode",))
    shape = tuple(eng.dims) if n == eng.N else (n,)
    return _prim_from_raw(out, shape, eng.ns, like)


def cons_to_prim(q, model, eps_neg: float = EPS_NEG) -> CellPrimitive:
    """Decode conservatives on the GPU (mixture.py:287-307)."""
    from .device import get_engine, is_torch
    if eps_neg != EPS_NEG:
        raise ValueError("the device decode uses the reference's eps_neg = 1e-10")
    eng = get_engine(None, model)
    qa = q if is_torch(q) else np.asarray(q, dtype=float)
    shape = tuple(qa.shape[:-1])
    n = int(np.prod(shape)) if shape else 1
    qs = eng.to_soa(qa.reshape(n, eng.nv), eng.nv)
    out = eng.empty(12 + eng.ns, n)
    eng._chk(eng.lib.csb_cons_to_prim(eng.ctx, n, qs.data_ptr(), out.data_ptr(),
                                      ctypes.c_void_p(eng.stream)), "cons_to_prim")
    eng.check("cons_to_prim", order=("decode",))
    prim = _prim_from_raw(out, shape, eng.ns, q)
    object.__setattr__(prim, "_q", q)
    return prim


def _primitive_call(model, rho, u, p, T, Y, want_prim, want_q):
    """One csb_primitive launch over the broadcast shape of the inputs."""
    from .device import get_engine, is_torch
    eng = get_engine(None, model)
    torch = eng.torch
    ns = eng.ns
    host = lambda x: None if x is None else (x.detach().cpu().numpy() if is_torch(x)
                                             else np.asarray(x, dtype=float))
    rho, p, T, u, Y = host(rho), host(p), host(T), host(u), host(Y)
    shapes = [np.shape(x) for x in (rho, p, T) if x is not None]
    shapes += [np.shape(u)[:-1], np.shape(Y)[:-1]]
    shape = tuple(np.broadcast_shapes(*shapes))
    n = int(np.prod(shape)) if shape else 1
    dev = lambda x, tail=(): (None if x is None else torch.from_numpy(
        np.array(np.broadcast_to(x, shape + tail), dtype=float).reshape(-1)).to(eng.device))
    tr, tp, tT = dev(rho), dev(p), dev(T)
    tu, tY = dev(u, (3,)), dev(Y, (ns,))
    out = eng.empty(12 + ns, n) if want_prim else None
    q = eng.empty(5 + ns, n) if want_q else None
    ptr = lambda t: t.data_ptr() if t is not None else None
    eng._chk(eng.lib.csb_primitive(eng.ctx, n, ptr(tr), ptr(tu), ptr(tp), ptr(tT), ptr(tY),
                                   ptr(out), ptr(q), ctypes.c_void_p(eng.stream)), "primitive")
    flags, _, _ = eng.status()
    if flags:
        raise NonPhysicalState("primitive state not admissible (rho, p and T must be > 0)")
    return eng, shape, out, q


def make_primitive(model, rho=None, u=(0.0, 0.0, 0.0), p=None, T=None, Y=None) -> CellPrimitive:
    """Consistent primitive state from two of (rho, p, T), u and Y, with
    p = rho R(Y) T (mixture.py:326-351); evaluated on the device."""
    if Y is None:
        raise ValueError("make_primitive needs the mass fractions Y")
    Ya = np.asarray(Y, dtype=float)
    if Ya.ndim == 1 and abs(float(Ya.sum()) - 1.0) > 1e-8:
        raise NonPhysicalState(f"mass fractions sum to {float(Ya.sum())!r}, not 1")
    if sum(x is not None for x in (rho, p, T)) < 2:
        raise ValueError("make_primitive needs two of rho, p, T")
    eng, shape, out, _ = _primitive_call(model, rho, u, p, T, Ya, True, False)
    prim = _prim_from_raw(out, shape, eng.ns, None)
    return CellPrimitive(**{k: v for k, v in vars(prim).items() if not k.startswith("_")})


def prim_to_cons(prim: CellPrimitive, model):
    """Conservative vector [rho, rho u, rho e_t, rho Y] (mixture.py:310-323),
    encoded on the device."""
    from .device import is_torch
    like = prim.rho if is_torch(prim.rho) else None
    eng, shape, _, q = _primitive_call(model, prim.rho, prim.u, None, prim.T, prim.Y, False, True)
    if like is not None:
        return q.t().reshape(shape + (eng.nv,)).to(like.device)
    return np.ascontiguousarray(q.t().cpu().numpy()).reshape(shape + (eng.nv,))


__all__ = ["R_UNIVERSAL", "EPS_NEG", "SpeciesData", "MixtureModel", "CellPrimitive",
           "species_table", "cons_to_prim", "make_primitive", "prim_to_cons", "padded_vector"]
