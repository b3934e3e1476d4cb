"""Finite-rate chemistry: mechanism description (host) and device evaluation.

Mirrors reference chemistry.py:21-104: ``Reaction``/``Mechanism`` data types,
``production_rates`` (mass-action Arrhenius), ``source_jacobian`` (central
finite differences with T frozen) and ``source_spectral_radius``.  The two
evaluators run on the GPU (csrc/csb_implicit.cuh); the mechanism file parser
is setup I/O and out of scope.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .device import get_engine, is_torch
from .errors import ValidationError


@dataclass(frozen=True)
class Reaction:
    """One elementary reaction (chemistry.py:21-37)."""

    reactant_stoich: np.ndarray
    product_stoich: np.ndarray
    A_f: float
    b_f: float
    Ea_f: float
    backward: Optional[Tuple[float, float, float]] = None

    def validate_mass_balance(self, model):
        lhs = float(np.asarray(self.reactant_stoich) @ model.M)
        rhs = float(np.asarray(self.product_stoich) @ model.M)
        if abs(lhs - rhs) > 1e-12 * max(lhs, rhs):
            raise ValidationError(
                [f"reaction does not conserve mass: {lhs:.15g} kg/mol vs {rhs:.15g} kg/mol"])


@dataclass(frozen=True)
class Mechanism:
    reactions: tuple
    enabled: bool = True


def _prepare(prim, mech, model):
    from .implicit import _q_of
    eng = get_engine(None, model)
    eng.set_mechanism(mech)
    q = _q_of(prim, model)
    qa = q if is_torch(q) else np.asarray(q, dtype=float)
    shape = tuple(qa.shape[:-1])
    n = int(np.prod(shape)) if shape else 1
    qs = eng.to_soa(qa.reshape(n, model.nvar), model.nvar)
    return eng, q, qs, shape, n


def production_rates(prim, mech: Optional[Mechanism], model):
    """Net chemical production per species, kg/(m^3 s) (chemistry.py:68-73)."""
    eng, q, qs, shape, n = _prepare(prim, mech, model)
    out = eng.empty(model.ns, n)
    eng._chk(eng.lib.csb_production_rates(eng.ctx, n, qs.data_ptr(), out.data_ptr(),
                                          ctypes.c_void_p(eng.stream)), "production_rates")
    eng.check("production_rates", order=("decode",))
    return eng.from_soa(out, q, shape + (model.ns,))


def source_jacobian(prim, mech: Optional[Mechanism], model):
    """d omega_s / d rho_r (1/s), shape (..., ns, ns) (chemistry.py:76-99)."""
    eng, q, qs, shape, n = _prepare(prim, mech, model)
    ns = model.ns
    out = eng.empty(ns * ns, n)
    eng._chk(eng.lib.csb_source_jacobian(eng.ctx, n, qs.data_ptr(), out.data_ptr(), None,
                                         ctypes.c_void_p(eng.stream)), "source_jacobian")
    eng.check("source_jacobian", order=("decode",))
    return eng.from_soa(out, q, shape + (ns * ns,)).reshape(shape + (ns, ns))


def source_spectral_radius(dOmega):
    """Row-sum bound max_s sum_r |dOmega_sr| (chemistry.py:102-104)."""
    if is_torch(dOmega):
        return dOmega.abs().sum(dim=-1).amax(dim=-1)
    return np.max(np.sum(np.abs(dOmega), axis=-1), axis=-1)


__all__ = ["Reaction", "Mechanism", "production_rates", "source_jacobian",
           "source_spectral_radius"]
