"""Mixture description and host-side state encoding.

Mirrors the data types and setup helpers of the reference ``csflow.mixture``
(reference mixture.py:33-104 SpeciesData/MixtureModel, 216-232 CellPrimitive,
310-351 prim_to_cons/make_primitive, 416-425 nitrogen_like/cloned_mixture).
These run once per case to build the freestream and the initial field.  The
per-iteration decode ``cons_to_prim`` runs on the GPU (``cons_to_prim``
below calls the CUDA library).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import NonPhysicalState

R_UNIVERSAL = 8.314462618  # J/(mol K), mixture.py:26
EPS_NEG = 1e-10            # mixture.py:30


@dataclass(frozen=True)
class SpeciesData:
    """Constant-cp species with Sutherland viscosity (mixture.py:33-55)."""

    name: str
    M: float
    cp: float
    hf: float
    Tref: float
    mu_ref: float
    T_mu: float
    S_mu: float

    def __post_init__(self):
        if self.M <= 0.0:
            raise ValueError(f"species {self.name}: molar mass must be positive")
        if self.cp <= R_UNIVERSAL / self.M:
            raise ValueError(f"species {self.name}: cp must exceed R_u/M (cv > 0)")
        if self.mu_ref < 0.0:
            raise ValueError(f"species {self.name}: mu_ref must be >= 0")


@dataclass(frozen=True)
class MixtureModel:
    """Ordered species plus Prandtl/Schmidt numbers (mixture.py:58-104)."""

    species: tuple
    Pr: float
    Sc: float
    M: np.ndarray = field(init=False, repr=False, compare=False)
    cp_s: np.ndarray = field(init=False, repr=False, compare=False)
    hf_s: np.ndarray = field(init=False, repr=False, compare=False)
    Tref_s: np.ndarray = field(init=False, repr=False, compare=False)
    R_s: np.ndarray = field(init=False, repr=False, compare=False)
    b_s: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        if len(self.species) < 1:
            raise ValueError("mixture needs at least one species")
        if self.Pr <= 0.0 or self.Sc <= 0.0:
            raise ValueError("Pr and Sc must be positive")
        names = [s.name for s in self.species]
        if len(set(names)) != len(names):
            raise ValueError("species names must be unique")
        col = lambda k: np.asarray([getattr(s, k) for s in self.species], dtype=float)
        object.__setattr__(self, "M", col("M"))
        object.__setattr__(self, "cp_s", col("cp"))
        object.__setattr__(self, "hf_s", col("hf"))
        object.__setattr__(self, "Tref_s", col("Tref"))
        object.__setattr__(self, "R_s", R_UNIVERSAL / self.M)
        object.__setattr__(self, "b_s", self.hf_s - self.cp_s * self.Tref_s)

    @property
    def ns(self) -> int:
        return len(self.species)

    @property
    def nvar(self) -> int:
        return 5 + self.ns

    def species_index(self, name: str) -> int:
        for i, s in enumerate(self.species):
            if s.name == name:
                return i
        raise KeyError(f"unknown species {name!r}")

    def table(self):
        """Per-species columns in the order the C-ABI expects."""
        col = lambda k: np.ascontiguousarray([getattr(s, k) for s in self.species], dtype=float)
        return {k: col(k) for k in ("M", "cp", "hf", "Tref", "mu_ref", "T_mu", "S_mu")}


@dataclass(frozen=True)
class CellPrimitive:
    """Decoded primitive state (mixture.py:216-232)."""

    rho: np.ndarray
    u: np.ndarray
    p: np.ndarray
    T: np.ndarray
    Y: np.ndarray
    c: np.ndarray
    gamma: np.ndarray
    h: np.ndarray
    Ek: np.ndarray


def mixture_gas_constant(Y, model: MixtureModel):
    return np.asarray(Y, dtype=float) @ model.R_s


def make_primitive(model: MixtureModel, rho=None, u=(0.0, 0.0, 0.0), p=None, T=None,
                   Y=None) -> CellPrimitive:
    """Consistent primitive state from two of (rho, p, T) plus Y (mixture.py:326-351)."""
    Y = np.asarray(Y, dtype=float)
    if Y.ndim == 1 and abs(float(np.sum(Y)) - 1.0) > 1e-8:
        raise NonPhysicalState("mass fractions must sum to 1")
    R = mixture_gas_constant(Y, model)
    if rho is None:
        rho = p / (R * T)
    elif T is None:
        T = p / (rho * R)
    elif p is None:
        p = rho * R * T
    rho = np.asarray(rho, dtype=float)
    T = np.asarray(T, dtype=float)
    p = np.asarray(p, dtype=float)
    u = np.broadcast_to(np.asarray(u, dtype=float), rho.shape + (3,)).copy()
    if np.any(rho <= 0) or np.any(T <= 0) or np.any(p <= 0):
        raise NonPhysicalState("freestream/primitive state not admissible")
    Y = np.broadcast_to(Y, rho.shape + (model.ns,)).copy()
    Ek = 0.5 * np.sum(u * u, axis=-1)
    cp = Y @ model.cp_s
    cv = cp - R
    gamma = cp / cv
    return CellPrimitive(rho=rho, u=u, p=p, T=T, Y=Y, c=np.sqrt(gamma * R * T), gamma=gamma,
                         h=Y @ model.b_s + cp * T + Ek, Ek=Ek)


def prim_to_cons(prim: CellPrimitive, model: MixtureModel):
    """Conservative vector [rho, rho u, rho e_t, rho Y] (mixture.py:310-323)."""
    rho = np.asarray(prim.rho, dtype=float)
    u = np.asarray(prim.u, dtype=float)
    Y = np.asarray(prim.Y, dtype=float)
    T = np.asarray(prim.T, dtype=float)
    Ek = 0.5 * np.sum(u * u, axis=-1)
    e_t = Y @ model.b_s + (Y @ model.cp_s) * T - (Y @ model.R_s) * T + Ek
    q = np.empty(rho.shape + (model.nvar,))
    q[..., 0] = rho
    q[..., 1:4] = rho[..., np.newaxis] * u
    q[..., 4] = rho * e_t
    q[..., 5:] = rho[..., np.newaxis] * Y
    return q


def padded_vector(prim: CellPrimitive, ns: int):
    """[rho, u, v, w, p, Y.., T] of a single state (fields.py:31-36 layout)."""
    return np.concatenate([np.atleast_1d(np.asarray(prim.rho, dtype=float)).reshape(1),
                           np.asarray(prim.u, dtype=float).reshape(3),
                           np.atleast_1d(np.asarray(prim.p, dtype=float)).reshape(1),
                           np.asarray(prim.Y, dtype=float).reshape(ns),
                           np.atleast_1d(np.asarray(prim.T, dtype=float)).reshape(1)])


def nitrogen_like(name: str = "N2") -> SpeciesData:
    """mixture.py:416-419."""
    return SpeciesData(name=name, M=0.028, cp=1039.0, hf=0.0, Tref=0.0,
                       mu_ref=1.663e-5, T_mu=273.15, S_mu=107.0)


def cloned_mixture(ns: int, Pr: float = 0.72, Sc: float = 0.7) -> MixtureModel:
    """mixture.py:422-425 (the paper's species-scaling benchmark mixture)."""
    return MixtureModel(species=tuple(nitrogen_like(f"N2_{i:04d}") for i in range(ns)),
                        Pr=Pr, Sc=Sc)


# ----------------------------------------------------------------------------
# device decode (cons_to_prim on the GPU)
# ----------------------------------------------------------------------------

class DevicePrimitive(CellPrimitive):
    """CellPrimitive produced on the device; keeps the conservative field so
    downstream device calls (cell_spectral_radii, ...) need not re-encode."""


def _decode_soa(eng, qs, like, n=None):
    """Device decode of SoA q (nv, N) -> CellPrimitive shaped like the grid
    (numpy unless `like` is a torch tensor)."""
    import ctypes
    n = eng.N if n is None else n
    out = eng.empty(12 + eng.ns, n)
    eng._chk(eng.lib.csb_cons_to_prim(eng.ctx, n, qs.data_ptr(), out.data_ptr(),
                                      ctypes.c_void_p(eng.stream)), "cons_to_prim")
    eng.check("cons_to_prim", order=("decode",))
    shape = tuple(eng.dims) if n == eng.N else (n,)
    return _prim_from_raw(out, shape, eng.ns, like)


def _prim_from_raw(out, shape, ns, like):
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


def cons_to_prim(q, model: MixtureModel, eps_neg: float = EPS_NEG) -> CellPrimitive:
    """Decode conservatives on the GPU (mixture.py:287-307)."""
    from .device import get_engine, is_torch
    if eps_neg != EPS_NEG:
        raise ValueError("the device decode uses the reference's eps_neg = 1e-10")
    eng = get_engine(None, model)
    qa = q if is_torch(q) else np.asarray(q, dtype=float)
    shape = tuple(qa.shape[:-1])
    n = int(np.prod(shape)) if shape else 1
    qs = eng.to_soa(qa.reshape(n, model.nvar), model.nvar)
    import ctypes
    out = eng.empty(12 + eng.ns, n)
    eng._chk(eng.lib.csb_cons_to_prim(eng.ctx, n, qs.data_ptr(), out.data_ptr(),
                                      ctypes.c_void_p(eng.stream)), "cons_to_prim")
    eng.check("cons_to_prim", order=("decode",))
    prim = _prim_from_raw(out, shape, model.ns, q)
    object.__setattr__(prim, "_q", q)
    return prim


def transport(prim: CellPrimitive, model: MixtureModel):
    """Mixture (mu, k, D) (mixture.py:354-372), evaluated on the host.

    Setup/diagnostic helper only (wall heat flux, tests); the kernels carry
    their own device copy of this closure."""
    T = np.asarray(prim.T, dtype=float)[..., np.newaxis]
    mu_ref = np.array([s.mu_ref for s in model.species])
    T_mu = np.array([s.T_mu for s in model.species])
    S_mu = np.array([s.S_mu for s in model.species])
    mu_s = mu_ref * (T / T_mu) ** 1.5 * (T_mu + S_mu) / (T + S_mu)
    mu = np.sum(np.asarray(prim.Y) * mu_s, axis=-1)
    k = mu * (np.asarray(prim.Y) @ model.cp_s) / model.Pr
    D = (mu / (np.asarray(prim.rho) * model.Sc))[..., np.newaxis] * np.ones(model.ns)
    return mu, k, D
