"""Build product (paper_2403_03440_b200) objects from golden fixtures or
config specs, plus the matching oracle objects."""

import numpy as np

import oracle as O
from golden_cases import KINDS, get, has
from paper_2403_03440_b200 import configs as C
from paper_2403_03440_b200.boundary import BoundaryCondition
from paper_2403_03440_b200.chemistry import Mechanism, Reaction
from paper_2403_03440_b200.grid import compute_metrics
from paper_2403_03440_b200.mixture import MixtureModel, SpeciesData, make_primitive

FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


def model_from_table(sp, PrSc):
    return MixtureModel(species=tuple(SpeciesData(f"S{i}", *map(float, row))
                                      for i, row in enumerate(sp)), Pr=float(PrSc[0]),
                        Sc=float(PrSc[1]))


def golden_product(case):
    """(grid, model, bcs, mech, q, cfl) for a golden case."""
    model = model_from_table(get(case, "species"), get(case, "PrSc"))
    grid = compute_metrics(get(case, "nodes"))
    kinds, tw, ax, fs = (get(case, k) for k in ("bc_kind", "bc_Twall", "bc_axis", "bc_fs"))
    bcs = {}
    for f, name in enumerate(FACES):
        kind = KINDS[int(kinds[f])]
        fr = None
        if kind == "farfield":
            v = fs[f]
            fr = make_primitive(model, rho=v[0], u=v[1:4], T=v[4], Y=v[5:])
        bcs[name] = BoundaryCondition(kind, freestream=fr,
                                      T_wall=None if np.isnan(tw[f]) else float(tw[f]),
                                      axis=None if ax[f] < 0 else int(ax[f]))
    mech = None
    if has(case, "rx_f"):
        nr, npd, fw, bw = (get(case, k) for k in ("rx_nu_r", "rx_nu_p", "rx_f", "rx_b"))
        mech = Mechanism(tuple(Reaction(nr[r], npd[r], *map(float, fw[r]),
                                        backward=None if np.isnan(bw[r][0]) else tuple(map(float, bw[r])))
                               for r in range(len(fw))))
    return grid, model, bcs, mech, get(case, "q"), float(get(case, "cfl"))


def spec_product(spec):
    """Product objects for a configs.CaseSpec."""
    model = MixtureModel(species=tuple(SpeciesData(s.name, s.M, s.cp, s.hf, s.Tref, s.mu_ref,
                                                   s.T_mu, s.S_mu) for s in spec.species),
                         Pr=spec.Pr, Sc=spec.Sc)
    grid = compute_metrics(spec.nodes)
    bcs = {}
    for name in FACES:
        b = spec.bcs[name]
        fr = None
        if b.fs is not None:
            rho, u, T, Y = b.fs
            fr = make_primitive(model, rho=rho, u=u, T=T, Y=Y)
        bcs[name] = BoundaryCondition(b.kind, freestream=fr, T_wall=b.T_wall, axis=b.axis)
    mech = None
    if spec.reactions:
        mech = Mechanism(tuple(Reaction(np.asarray(r.nu_r, float), np.asarray(r.nu_p, float), r.Af,
                                        r.bf, r.Eaf, backward=r.back) for r in spec.reactions))
    return grid, model, bcs, mech


def spec_oracle(spec):
    th = O.Thermo([s.M for s in spec.species], [s.cp for s in spec.species],
                  [s.hf for s in spec.species], [s.Tref for s in spec.species],
                  [s.mu_ref for s in spec.species], [s.T_mu for s in spec.species],
                  [s.S_mu for s in spec.species], spec.Pr, spec.Sc)
    grid = O.Grid(spec.nodes)
    bcs = {}
    for name in FACES:
        b = spec.bcs[name]
        vec = None
        if b.fs is not None:
            rho, u, T, Y = b.fs
            vec = O.freestream_vector(rho, u, T, Y, th)
        bcs[name] = O.BC(b.kind, fs=vec, Tw=b.T_wall, axis=b.axis)
    mech = None
    if spec.reactions:
        mech = O.Mech(tuple(O.Rx(np.asarray(r.nu_r, float), np.asarray(r.nu_p, float), r.Af, r.bf,
                                 r.Eaf, r.back) for r in spec.reactions))
    return th, grid, bcs, mech
