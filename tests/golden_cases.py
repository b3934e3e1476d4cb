"""Rebuild golden-fixture cases (tests/golden/golden.npz) as oracle objects."""

import os

import numpy as np

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
KINDS = ("farfield", "supersonic_outflow", "noslip_isothermal", "symmetry", "periodic")
_CACHE = {}


def load():
    if "z" not in _CACHE:
        z = np.load(GOLDEN)
        _CACHE["z"] = {k: z[k] for k in z.files}
    return _CACHE["z"]


def get(case, key):
    return load()[f"{case}/{key}"]


def has(case, key):
    return f"{case}/{key}" in load()


def thermo(case):
    sp = get(case, "species")
    Pr, Sc = get(case, "PrSc")
    return O.Thermo(*[sp[:, c] for c in range(7)], Pr=Pr, Sc=Sc)


def bcs(case, th):
    kinds = get(case, "bc_kind")
    tw = get(case, "bc_Twall")
    ax = get(case, "bc_axis")
    fs = get(case, "bc_fs")
    out = {}
    for f, name in enumerate(O.FACES):
        kind = KINDS[int(kinds[f])]
        vec = None
        if kind == "farfield":
            v = fs[f]
            vec = O.freestream_vector(v[0], v[1:4], v[4], v[5:], th)
        out[name] = O.BC(kind, fs=vec, Tw=None if np.isnan(tw[f]) else float(tw[f]),
                         axis=None if ax[f] < 0 else int(ax[f]))
    return out


def mech(case):
    if not has(case, "rx_f"):
        return None
    nr, npd, fw, bw = (get(case, k) for k in ("rx_nu_r", "rx_nu_p", "rx_f", "rx_b"))
    rs = tuple(O.Rx(nr[r], npd[r], *map(float, fw[r]),
                    back=None if np.isnan(bw[r][0]) else tuple(map(float, bw[r])))
               for r in range(len(fw)))
    return O.Mech(rs)


def grid(case):
    return O.Grid(get(case, "nodes"))


def relerr(a, b):
    """max |a-b| / max |b|, per trailing component when 4-D or more."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / den) if den > 0 else float(np.max(np.abs(a - b)))


def comp_relerr(a, b):
    """Worst over components c of max_cells |a-b| / max_cells |b|."""
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    a2 = a.reshape(-1, a.shape[-1])
    b2 = b.reshape(-1, b.shape[-1])
    worst = 0.0
    for c in range(a2.shape[1]):
        den = np.max(np.abs(b2[:, c]))
        num = np.max(np.abs(a2[:, c] - b2[:, c]))
        worst = max(worst, num / den if den > 0 else num)
    return worst
