"""LU-SGS forward/backward sweeps on the GPU (drop-in for reference
lusgs.py:250-274 ``lusgs_solve``).

The sweeps run on the device operator produced by ``assemble_lhs``: a
pipelined wavefront kernel for 2-D grids and hyperplane launches for 3-D
(csrc/csb_sweep.cuh, csrc/csb_wavefront.cuh).
"""

from __future__ import annotations

import ctypes

from .device import SoA, is_torch


def lusgs_solve(op, rhs, *, return_forward=False):
    """Forward/backward LU-SGS sweeps of the assembled operator; returns dQ.

    ``return_forward`` (extension for parity tests): also return dq*, the
    forward-sweep result the reference's ``_cs_forward``/``_ci_forward``
    leave in dq (lusgs.py:62-103, 150-197).
    """
    eng = op._eng
    op.ensure_current()
    rs = eng.to_soa(rhs, eng.nv)
    dq = eng.empty(eng.nv, eng.N)
    star = eng.empty(eng.nv, eng.N) if return_forward else None
    eng._chk(eng.lib.csb_lusgs(eng.ctx, rs.data_ptr(), dq.data_ptr(),
                               star.data_ptr() if star is not None else None,
                               ctypes.c_void_p(eng.stream)), "lusgs_solve")
    eng.check("lusgs_solve", order=("singular",))
    if isinstance(rhs, SoA):
        out = SoA(dq, eng.dims)
        return (out, SoA(star, eng.dims)) if return_forward else out
    like = rhs if is_torch(rhs) else op._like
    shape = tuple(eng.dims) + (eng.nv,)
    import numpy as np
    lk = like if like is not None else np.empty(0)
    out = eng.from_soa(dq, lk, shape)
    if return_forward:
        return out, eng.from_soa(star, lk, shape)
    return out


__all__ = ["lusgs_solve"]
