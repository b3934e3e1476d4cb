"""csflow-b200: B200-native implicit pseudo-time iteration of arXiv 2403.03440.

Drop-in for the reference ``csflow`` solver entry points (same names and
signatures); the compute runs in the sm_100a library
``paper_2403_03440_b200/_lib/libcsflow_b200.so`` through its C ABI
(include/csflow_b200.h).  There is no CPU fallback.
"""

from .boundary import BoundaryCondition  # noqa: F401
from .errors import (BadDims, CsflowError, DegenerateCell, Diverged, ExtensionMissing,  # noqa: F401
                     MissingBC, NonPhysicalState, NoWallBoundary, SingularDiagonal, ZeroWavespeed)
from .grid import StructuredGrid, compute_metrics, generate_box, generate_cylinder_ogrid  # noqa: F401
from .mixture import (CellPrimitive, MixtureModel, SpeciesData, cloned_mixture,  # noqa: F401
                      cons_to_prim, make_primitive, nitrogen_like, prim_to_cons)

__version__ = "0.1.0"


def library_path():
    from ._lib import LIB_PATH
    return LIB_PATH
