"""csflow-b200: B200-native implicit pseudo-time iteration of arXiv 2403.03440.

Drop-in for the reference ``csflow`` solver entry points (same names and
signatures); the compute runs in the sm_100a library
``paper_2403_03440_b200/_lib/libcsflow_b200.so`` through its C ABI
(include/csflow_b200.h).  There is no CPU fallback.
"""

from .boundary import BoundaryCondition  # noqa: F401
from .errors import (BadDims, CsflowError, DegenerateCell, Diverged, ExtensionMissing,  # noqa: F401
                     MissingBC, MultiBlockUnsupported, NonPhysicalState, NoWallBoundary,
                     ParseError, SingularDiagonal, ZeroWavespeed)
from .grid import StructuredGrid, compute_metrics, generate_box, generate_cylinder_ogrid  # noqa: F401
from .configs import cloned_mixture, nitrogen_like  # noqa: F401
from .mixture import (CellPrimitive, MixtureModel, SpeciesData, cons_to_prim,  # noqa: F401
                      make_primitive, prim_to_cons)
from .plot3d import read_plot3d, write_plot3d  # noqa: F401

__version__ = "0.1.0"


def library_path():
    from ._lib import LIB_PATH
    return LIB_PATH
