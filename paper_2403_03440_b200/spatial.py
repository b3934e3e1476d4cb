"""Explicit residual R (V dQ/dt = -R) on the GPU.

Drop-in for reference spatial.py:207-274 ``assemble_residual``: same
signature, same return (AoS ``(ni, nj, nk, 5+ns)`` in the caller's array
flavour), same exceptions.  The work is one sm_100a kernel (csrc/csb_rhs.cuh):
decode + ghost fill + MUSCL/Rusanov + viscous + source, tile by tile.
"""

from __future__ import annotations

import ctypes

from .device import F_KSKIP, SoA, get_engine, is_torch


def residual_device(eng, qs, first_order=False, padded=False, R=None):
    """SoA in, SoA out: R (nv, N) [and P (6+ns, (ni+4)(nj+4)(nk+4))]."""
    ni, nj, nk = eng.dims
    R = eng.empty(eng.nv, eng.N) if R is None else R
    P = eng.empty(6 + eng.ns, (ni + 4) * (nj + 4) * (nk + 4)) if padded else None
    eng._chk(eng.lib.csb_residual(eng.ctx, qs.data_ptr(), R.data_ptr(),
                                  P.data_ptr() if P is not None else None,
                                  int(bool(first_order)), ctypes.c_void_p(eng.stream)),
             "residual")
    # F_KSKIP only records that the library re-ran the 2-D fast path's
    # tiles on the general path (w != 0 under symmetry k-faces); R is valid
    flags, cell, _ = eng.status()
    flags &= ~F_KSKIP
    if flags:
        eng.raise_for(flags, cell, "assemble_residual", order=("decode",))
    return R, P


def assemble_residual(q, grid, bcs, mech, model, *, first_order: bool = False,
                      return_padded: bool = False):
    """Assemble the extensive residual R on interior cells (spatial.py:207-274)."""
    eng = get_engine(grid, model)
    eng.set_bcs(bcs)
    eng.set_mechanism(mech)
    qs = eng.to_soa(q, eng.nv)
    R, P = residual_device(eng, qs, first_order, return_padded)
    if isinstance(q, SoA):
        out = SoA(R, eng.dims)
        return (out, SoA(P, tuple(n + 4 for n in eng.dims))) if return_padded else out
    Rout = eng.from_soa(R, q, tuple(eng.dims) + (eng.nv,))
    if not return_padded:
        return Rout
    ni, nj, nk = eng.dims
    Pout = eng.from_soa(P, q, (ni + 4, nj + 4, nk + 4, 6 + eng.ns))
    return Rout, Pout


__all__ = ["assemble_residual", "residual_device", "is_torch"]
