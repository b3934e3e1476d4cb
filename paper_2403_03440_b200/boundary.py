"""Boundary-condition descriptors (reference boundary.py:21-38).

The ghost fill itself runs on the GPU inside the residual kernel (it
reproduces the reference's face-by-face fill order, boundary.py:53-114,
including corner and NaN-ghost semantics).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .errors import MissingBC
from .mixture import CellPrimitive

FACE_NAMES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")
BC_KINDS = ("farfield", "supersonic_outflow", "noslip_isothermal", "symmetry", "periodic")


@dataclass(frozen=True)
class BoundaryCondition:
    kind: str
    freestream: Optional[CellPrimitive] = None
    T_wall: Optional[float] = None
    axis: Optional[int] = None

    def __post_init__(self):
        if self.kind not in BC_KINDS:
            raise MissingBC(f"unknown boundary kind {self.kind!r}")
        if self.kind == "farfield" and self.freestream is None:
            raise MissingBC("farfield boundary requires a freestream state")
        if self.kind == "noslip_isothermal" and (self.T_wall is None or self.T_wall <= 0):
            raise MissingBC("isothermal wall requires T_wall > 0")


def validate_bcs(bcs):
    """Presence and periodic pairing checks (boundary.py:60-70)."""
    for name in FACE_NAMES:
        if name not in bcs:
            raise MissingBC(f"no boundary condition for face {name!r}")
    for fid, name in enumerate(FACE_NAMES):
        if bcs[name].kind == "periodic":
            axis, side = divmod(fid, 2)
            opp = FACE_NAMES[axis * 2 + (1 - side)]
            if bcs[opp].kind != "periodic":
                raise MissingBC(f"periodic face {name!r} requires periodic {opp!r}")
