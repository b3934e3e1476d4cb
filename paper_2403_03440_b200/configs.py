"""Seeded synthetic inputs for BASELINE.json configs 0-4.

No public dataset is involved: BASELINE.json's configs define the inputs.
Everything is drawn from one ``numpy.random.default_rng(seed)`` per case in
a documented order, so the GPU and the CPU oracle see identical arrays.

Documented choices:
* single temperature: the reference has no T_v; T_v is still drawn so the RNG
  stream is as specified, then discarded (G1);
* 5-species air uses the reference's ``air5_model`` test thermo
  (pkg/tests/conftest.py:22-34); no rate data ships, so chemistry is frozen
  unless a synthetic mechanism is requested (G2);
* 11-species ionised air uses builder-authored constant-cp thermo (molar
  masses of the named species, cp/R = 3.5 molecules / 2.5 atoms+electron,
  hf from air5 for neutrals and 0 for ions) (G3);
* synthetic species/mechanisms for ns=20/40 follow the config-3 recipe;
* O-grids honour stretch 1.02 and wall spacing 1e-5 m literally, which fixes
  the outer radius at 1 + 1e-5 (1.02^nj - 1)/0.02 (G9);
* boxes use dz = 1e-3 m, outflow on i/j and symmetry on k; O-grids use the
  reference's cylinder_case BCs (pkg/tests/test_driver.py:108-123).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

R_U = 8.314462618

AIR5 = (  # name, M [kg/mol], cp [J/kg K], hf [J/kg]; Tref 298.15, mu 1.7e-5/273.15/110
    ("N2", 0.0280134, 1039.0, 0.0),
    ("O2", 0.0319988, 918.0, 0.0),
    ("NO", 0.0300061, 995.0, 3.0e6),
    ("N", 0.0140067, 1484.0, 3.36e7),
    ("O", 0.0159994, 1300.0, 1.54e7),
)

AIR11_MASS = (("N2", 0.0280134, 3.5), ("O2", 0.0319988, 3.5), ("NO", 0.0300061, 3.5),
              ("N", 0.0140067, 2.5), ("O", 0.0159994, 2.5), ("N2+", 0.0280129, 3.5),
              ("O2+", 0.0319983, 3.5), ("NO+", 0.0300056, 3.5), ("N+", 0.0140062, 2.5),
              ("O+", 0.0159989, 2.5), ("e-", 5.4858e-7, 2.5))

FACES = ("imin", "imax", "jmin", "jmax", "kmin", "kmax")


@dataclass
class SpeciesSpec:
    name: str
    M: float
    cp: float
    hf: float
    Tref: float
    mu_ref: float
    T_mu: float
    S_mu: float


@dataclass
class ReactionSpec:
    nu_r: np.ndarray
    nu_p: np.ndarray
    Af: float
    bf: float
    Eaf: float
    back: Optional[tuple] = None


@dataclass
class BCSpec:
    kind: str
    fs: Optional[tuple] = None     # (rho, (u, v, w), T, Y) freestream, make_primitive(rho,u,T,Y)
    T_wall: Optional[float] = None
    axis: Optional[int] = None


@dataclass
class CaseSpec:
    name: str
    nodes: np.ndarray
    species: list
    bcs: dict
    q: np.ndarray
    cfl: float
    Pr: float = 0.72
    Sc: float = 0.7
    reactions: Optional[list] = None
    scheme: str = "CS1"
    extra: dict = field(default_factory=dict)

    @property
    def dims(self):
        return tuple(int(n) - 1 for n in self.nodes.shape[:3])

    @property
    def ns(self):
        return len(self.species)

    @property
    def nv(self):
        return 5 + len(self.species)

    @property
    def ncells(self):
        a, b, c = self.dims
        return a * b * c


# ----------------------------------------------------------------- species

# Nitrogen-like species of the paper's species-scaling benchmark (reference
# mixture.py:416-425): M, cp, hf, Tref, mu_ref, T_mu, S_mu
NITROGEN_LIKE = (0.028, 1039.0, 0.0, 0.0, 1.663e-5, 273.15, 107.0)


def nitrogen_like(name: str = "N2"):
    from .mixture import SpeciesData
    return SpeciesData(name, *NITROGEN_LIKE)


def cloned_mixture(ns: int, Pr: float = 0.72, Sc: float = 0.7):
    """ns identical nitrogen-like species (the paper's scaling mixture)."""
    from .mixture import MixtureModel
    return MixtureModel([nitrogen_like(f"N2_{i:04d}") for i in range(ns)], Pr=Pr, Sc=Sc)


def air5_species():
    return [SpeciesSpec(n, M, cp, hf, 298.15, 1.7e-5, 273.15, 110.0) for n, M, cp, hf in AIR5]


def air11_species():
    hf5 = {n: hf for n, _, _, hf in AIR5}
    out = []
    for n, M, cpr in AIR11_MASS:
        out.append(SpeciesSpec(n, M, cpr * R_U / M, hf5.get(n, 0.0), 298.15 if n in hf5 else 0.0,
                               1.7e-5, 273.15, 110.0))
    return out


def synthetic_species(ns, rng):
    """Config-3 recipe: M ~ U(1,50) g/mol, cp/R ~ U(2.5,4.5), hf = Tref = 0,
    nitrogen-like Sutherland data (mixture.py:416-419)."""
    M = rng.uniform(1.0, 50.0, ns) * 1e-3
    cpr = rng.uniform(2.5, 4.5, ns)
    return [SpeciesSpec(f"S{s:02d}", float(M[s]), float(cpr[s] * R_U / M[s]), 0.0, 0.0,
                        1.663e-5, 273.15, 107.0) for s in range(ns)]


def synthetic_mechanism(ns, rng, n_reactions=None):
    """2*ns reversible A <-> B reactions among random species pairs;
    log10 A ~ U(10,18), b ~ U(-2,1), Ta ~ U(1e4,1e5) K for forward and
    backward rates independently; Ea = R_u Ta.  Not mass balanced (the
    reference validates balance only in its file parser, chemistry.py:181)."""
    nr = 2 * ns if n_reactions is None else n_reactions
    out = []
    for _ in range(nr):
        a, b = rng.choice(ns, size=2, replace=False) if ns > 1 else (0, 0)
        nu_r = np.zeros(ns)
        nu_p = np.zeros(ns)
        nu_r[a] = 1.0
        nu_p[b] = 1.0
        fw = (10.0 ** rng.uniform(10.0, 18.0), rng.uniform(-2.0, 1.0), R_U * rng.uniform(1e4, 1e5))
        bw = (10.0 ** rng.uniform(10.0, 18.0), rng.uniform(-2.0, 1.0), R_U * rng.uniform(1e4, 1e5))
        out.append(ReactionSpec(nu_r, nu_p, *fw, back=bw))
    return out


# ------------------------------------------------------------------- state

def _thermo_arrays(species):
    M = np.array([s.M for s in species])
    cp = np.array([s.cp for s in species])
    b = np.array([s.hf - s.cp * s.Tref for s in species])
    return M, cp, R_U / M, b


def encode_state(rho, u, T, Y, species):
    """prim_to_cons(make_primitive(rho=, u=, T=, Y=)) (mixture.py:310-351)."""
    _, cp, Rs, bs = _thermo_arrays(species)
    Ek = 0.5 * np.sum(u * u, axis=-1)
    e_t = Y @ bs + (Y @ cp) * T - (Y @ Rs) * T + Ek
    q = np.empty(rho.shape + (5 + len(species),))
    q[..., 0] = rho
    q[..., 1:4] = rho[..., np.newaxis] * u
    q[..., 4] = rho * e_t
    q[..., 5:] = rho[..., np.newaxis] * Y
    return q


def random_fields(dims, ns, rng):
    """Config-0 distributions, draw order rho, u, v, T, Tv, Y."""
    shp = tuple(dims)
    rho = 10.0 ** rng.uniform(-3.0, -1.0, shp)
    u = rng.uniform(-3000.0, 3000.0, shp)
    v = rng.uniform(-3000.0, 3000.0, shp)
    T = rng.uniform(300.0, 8000.0, shp)
    _tv = rng.uniform(300.0, 8000.0, shp)  # two-temperature slot: unused
    Y = rng.dirichlet(np.ones(ns), size=shp)
    vel = np.stack([u, v, np.zeros(shp)], axis=-1)
    return rho, vel, T, Y


def random_state(dims, species, rng, electron=None, smooth_sigma=None):
    rho, vel, T, Y = random_fields(dims, len(species), rng)
    if electron is not None:
        Y[..., electron] = np.minimum(Y[..., electron], 1e-8)
        Y = Y / np.sum(Y, axis=-1, keepdims=True)
    if smooth_sigma:
        from scipy.ndimage import gaussian_filter
        sm = lambda a: gaussian_filter(a, sigma=(smooth_sigma, smooth_sigma, 0), mode="nearest")
        rho, T = sm(rho), sm(T)
        vel = np.stack([sm(vel[..., c]) for c in range(3)], axis=-1)
        Y = np.stack([sm(Y[..., s]) for s in range(Y.shape[-1])], axis=-1)
        if electron is not None:
            Y[..., electron] = np.minimum(Y[..., electron], 1e-8)
        Y = Y / np.sum(Y, axis=-1, keepdims=True)
    return encode_state(rho, vel, T, Y, species)


# ------------------------------------------------------------------- grids

def box_nodes(extent, dims):
    dims = tuple(int(d) for d in dims)
    ext = np.broadcast_to(np.asarray(extent, dtype=float), (3,))
    axes = [np.linspace(0.0, ext[d], dims[d] + 1) for d in range(3)]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


def ogrid_outer_radius(nj, wall=1e-5, stretch=1.02, radius=1.0):
    return radius + wall * (stretch ** nj - 1.0) / (stretch - 1.0)


def ogrid_nodes(dims, stretch=1.02, wall=1e-5, radius=1.0):
    """generate_cylinder_ogrid(1, R_out, dims, stretch=1.02) (grid.py:139-162)."""
    ni, nj, nk = dims
    outer = ogrid_outer_radius(nj, wall, stretch, radius)
    th = np.deg2rad(np.linspace(270.0, 90.0, ni + 1))
    L = outer - radius
    h0 = L * (stretch - 1.0) / (stretch ** nj - 1.0)
    r = radius + np.concatenate(([0.0], np.cumsum(h0 * stretch ** np.arange(nj))))
    z = np.linspace(0.0, 0.1 * radius, nk + 1)
    nodes = np.empty((ni + 1, nj + 1, nk + 1, 3))
    nodes[..., 0] = (r[np.newaxis, :] * np.cos(th)[:, np.newaxis])[..., np.newaxis]
    nodes[..., 1] = (r[np.newaxis, :] * np.sin(th)[:, np.newaxis])[..., np.newaxis]
    nodes[..., 2] = z[np.newaxis, np.newaxis, :]
    return nodes


def box_bcs():
    return {"imin": BCSpec("supersonic_outflow"), "imax": BCSpec("supersonic_outflow"),
            "jmin": BCSpec("supersonic_outflow"), "jmax": BCSpec("supersonic_outflow"),
            "kmin": BCSpec("symmetry"), "kmax": BCSpec("symmetry")}


def cylinder_bcs(fs, T_wall=300.0):
    return {"imin": BCSpec("supersonic_outflow"), "imax": BCSpec("supersonic_outflow"),
            "jmin": BCSpec("noslip_isothermal", T_wall=T_wall), "jmax": BCSpec("farfield", fs=fs),
            "kmin": BCSpec("symmetry"), "kmax": BCSpec("symmetry")}


def freestream_air11(rng):
    """Config 4: 1e-3 kg/m^3, 6000 m/s, 300 K, Y from seed normalised (electron
    capped at 1e-8 as in config 2)."""
    Y = rng.uniform(0.0, 1.0, 11)
    Y[10] = min(Y[10], 1e-8)
    Y = Y / Y.sum()
    return (1e-3, (6000.0, 0.0, 0.0), 300.0, Y)


# ----------------------------------------------------------------- configs

def config0(seed=0, dims=(64, 64, 1), cfl=10.0):
    rng = np.random.default_rng(seed)
    sp = air5_species()
    d = (int(dims[0]), int(dims[1]), 1)
    return CaseSpec("config0", box_nodes((1e-3 * d[0], 1e-3 * d[1], 1e-3), d), sp, box_bcs(),
                    random_state(d, sp, rng), cfl)


def config1(seed=1, dims=(512, 512, 1), cfl=50.0):
    c = config0(seed, dims, cfl)
    c.name = "config1"
    return c


def config2(seed=2, dims=(1024, 1024, 1), cfl=100.0, sigma=4.0):
    rng = np.random.default_rng(seed)
    sp = air11_species()
    fs = freestream_air11(np.random.default_rng(seed + 1000))
    q = random_state(dims, sp, rng, electron=10, smooth_sigma=sigma)
    return CaseSpec("config2", ogrid_nodes(dims), sp, cylinder_bcs(fs), q, cfl,
                    extra={"iterations": 10})


def config3(ns, seed=3, dims=(1024, 1024, 1), cfl=10.0, chemistry=False):
    rng = np.random.default_rng(seed + ns)
    if ns == 5:
        sp = air5_species()
    elif ns == 11:
        sp = air11_species()
    else:
        sp = synthetic_species(ns, rng)
    rx = synthetic_mechanism(ns, rng) if chemistry else None
    d = tuple(int(x) for x in dims)
    q = random_state(d, sp, rng)
    return CaseSpec(f"config3_ns{ns}", box_nodes((1e-3 * d[0], 1e-3 * d[1], 1e-3), d), sp,
                    box_bcs(), q, cfl, reactions=rx)


def config4(seed=4, dims=(4096, 2048, 1)):
    rng = np.random.default_rng(seed)
    sp = air11_species()
    fs = freestream_air11(rng)
    rho, vel, T, Y = fs
    q0 = encode_state(np.asarray(rho), np.asarray(vel, dtype=float), np.asarray(T), Y, sp)
    q = np.broadcast_to(q0, tuple(dims) + (16,)).copy()  # Case.initial_field (driver.py:67-69)
    return CaseSpec("config4", ogrid_nodes(dims), sp, cylinder_bcs(fs), q, 1000.0,
                    extra={"iterations": 500, "cfl_ramp": (1.0, 2.0, 45)})


# ------------------------------------------------------------ product objects

def model_of(spec):
    from .mixture import MixtureModel, SpeciesData
    return MixtureModel([SpeciesData(s.name, s.M, s.cp, s.hf, s.Tref, s.mu_ref, s.T_mu, s.S_mu)
                         for s in spec.species], Pr=spec.Pr, Sc=spec.Sc)


def build_case(spec):
    """(grid, model, bcs, mech) drop-in objects for a CaseSpec."""
    from .boundary import BoundaryCondition
    from .chemistry import Mechanism, Reaction
    from .grid import compute_metrics
    from .mixture import make_primitive
    model = model_of(spec)
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


def freestream_of(spec, model):
    """The freestream ``CellPrimitive`` of a case with a far-field boundary
    (``Case.freestream``), else the first cell's state."""
    from .mixture import make_primitive
    for b in spec.bcs.values():
        if b.fs is not None:
            rho, u, T, Y = b.fs
            return make_primitive(model, rho=rho, u=u, T=T, Y=Y)
    q = spec.q.reshape(-1, spec.nv)[0]
    Y = q[5:] / q[0]
    M, cp, Rs, bs = _thermo_arrays(spec.species)
    u = q[1:4] / q[0]
    T = (q[4] / q[0] - 0.5 * u @ u - Y @ bs) / (Y @ cp - Y @ Rs)
    return make_primitive(model, rho=q[0], u=u, T=T, Y=Y)
