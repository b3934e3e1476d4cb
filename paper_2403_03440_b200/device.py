"""Device-side state of one case: the C-ABI context, uploaded grid metrics,
mechanism, boundary conditions and the workspace (PyTorch device buffers).

Every public API function of the package resolves its (grid, model) pair to
an ``Engine`` (cached), converts reference-layout arrays (AoS
``(ni, nj, nk, comp)``, numpy or torch) to the library's SoA layout with the
library's own transpose kernel, calls the C ABI, and maps the device flag
word back onto the reference's exception classes.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .boundary import BC_KINDS, FACE_NAMES, validate_bcs
from .errors import (DeviceError, ExtensionMissing, MissingBC, NonPhysicalState,
                     SingularDiagonal, ZeroWavespeed)
from .mixture import padded_vector, species_table

F_DECODE, F_FACE_T, F_RES_NONFINITE, F_ZERO_WAVE = 1, 2, 4, 8
F_SINGULAR, F_GATE, F_KSKIP, F_BLOCK, F_GATE_DECODE = 16, 32, 64, 128, 256
SCHEMES = {"CI": 0, "CS1": 1, "CS2": 2}
OP_FIELDS = {"w": 0, "b": 1, "sp_lower": 2, "sp_upper": 3, "d_scal": 4, "d_species": 5,
             "lam_face0": 6, "lam_face1": 7, "lam_face2": 8, "lam_face_sp0": 9,
             "lam_face_sp1": 10, "lam_face_sp2": 11, "dinv": 12, "vdom": 13}


def torch_mod():
    try:
        import torch
    except Exception as exc:  # pragma: no cover
        raise ExtensionMissing(f"torch is required for device buffers: {exc}")
    return torch


def require_cuda():
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: csflow-b200 runs only on the GPU (sm_100a); "
                               "there is no CPU fallback")
    return torch


class Engine:
    """One C-ABI context bound to a grid and a mixture model."""

    def __init__(self, grid, model, device=None):
        torch = require_cuda()
        self.torch = torch
        self.lib = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        if grid is None:  # grid-free engine: model, mechanism and flags only
            grid = _unit_grid(self.device)
        self.grid = grid
        self.model = model
        self.ns = len(model.species)
        self.nv = 5 + self.ns
        self.dims = tuple(grid.dims)
        self.N = int(np.prod(self.dims))
        ctx = ctypes.c_void_p()
        self._chk(self.lib.csb_create(ctypes.byref(ctx)), "create")
        self.ctx = ctx
        tab = species_table(model)
        self._keep = [tab]
        self._chk(self.lib.csb_set_model(ctx, self.ns, *[_lib.hp(tab[k]) for k in
                                                         ("M", "cp", "hf", "Tref", "mu_ref",
                                                          "T_mu", "S_mu")],
                                         float(model.Pr), float(model.Sc)), "set_model")
        dm = getattr(grid, "device_metrics", None)
        if callable(dm):  # this package's grids: metrics already on the device
            S, vol = dm(self.device)
            self.S, self.vol = list(S), vol
        else:  # any grid with the reference's attributes (duck typing)
            soa = lambda a: torch.from_numpy(
                np.ascontiguousarray(np.moveaxis(np.asarray(a, float), -1, 0).reshape(3, -1))
            ).to(self.device)
            self.S = [soa(grid.Si), soa(grid.Sj), soa(grid.Sk)]
            self.vol = torch.from_numpy(np.ascontiguousarray(grid.volume, dtype=float).reshape(-1)
                                        ).to(self.device)
        ni, nj, nk = self.dims
        self._chk(self.lib.csb_set_grid(ctx, ni, nj, nk, *[t.data_ptr() for t in self.S],
                                        self.vol.data_ptr()), "set_grid")
        self._mech = ()
        self._bcs = None
        self.ws = None
        self.ws_block = False
        self.set_mechanism(None)
        self.ensure_workspace(False)

    def __del__(self):
        try:
            if getattr(self, "ctx", None) is not None:
                self.lib.csb_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # ----------------------------------------------------------------- plumbing
    def _chk(self, rc, what):
        if rc == 0:
            return
        msg = ""
        if getattr(self, "ctx", None) is not None:
            raw = self.lib.csb_last_error(self.ctx)
            msg = raw.decode() if raw else ""
        if rc == 5:
            raise MissingBC(msg)
        raise DeviceError(f"{what} failed (code {rc}): {msg}")

    @property
    def stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device=self.device)

    def zeros(self, *shape):
        return self.torch.zeros(*shape, dtype=self.torch.float64, device=self.device)

    def ensure_workspace(self, with_block):
        if self.ws is not None and (self.ws_block or not with_block):
            return
        nbytes = self.lib.csb_workspace_bytes(self.ctx, 1 if with_block else 0)
        self.ws = self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.device)
        self._chk(self.lib.csb_set_workspace(self.ctx, self.ws.data_ptr(), int(nbytes)),
                  "set_workspace")
        self.ws_block = bool(with_block)

    def set_mechanism(self, mech):
        if mech is self._mech:
            return
        ns = self.ns
        if mech is None or not mech.reactions:
            z = np.zeros(1)
            self._chk(self.lib.csb_set_mechanism(self.ctx, 0, _lib.hp(z), _lib.hp(z), _lib.hp(z),
                                                 _lib.hp(z), 0), "set_mechanism")
        else:
            rx = mech.reactions
            nu_r = np.ascontiguousarray([np.asarray(r.reactant_stoich, float) for r in rx])
            nu_p = np.ascontiguousarray([np.asarray(r.product_stoich, float) for r in rx])
            fw = np.ascontiguousarray([[r.A_f, r.b_f, r.Ea_f] for r in rx], dtype=float)
            bw = np.ascontiguousarray([list(r.backward) if r.backward is not None
                                       else [np.nan] * 3 for r in rx], dtype=float)
            assert nu_r.shape == (len(rx), ns)
            self._chk(self.lib.csb_set_mechanism(self.ctx, len(rx), _lib.hp(nu_r), _lib.hp(nu_p),
                                                 _lib.hp(fw), _lib.hp(bw), int(bool(mech.enabled))),
                      "set_mechanism")
        self._mech = mech

    def chem_on(self):
        m = self._mech
        return m is not None and bool(getattr(m, "enabled", False)) and bool(m.reactions)

    def set_bcs(self, bcs):
        if bcs is self._bcs:
            return
        validate_bcs(bcs)
        for f, name in enumerate(FACE_NAMES):
            bc = bcs[name]
            kind = BC_KINDS.index(bc.kind)
            fs = None
            if bc.kind == "farfield":
                fs = np.ascontiguousarray(padded_vector(bc.freestream, self.ns))
                self._keep.append(fs)
            self._chk(self.lib.csb_set_bc(self.ctx, f, kind,
                                          float(bc.T_wall) if bc.T_wall is not None else 0.0,
                                          -1 if bc.axis is None else int(bc.axis),
                                          _lib.hp(fs) if fs is not None else None), "set_bc")
        self._bcs = bcs

    def status(self):
        fl = ctypes.c_ulonglong()
        cell = ctypes.c_longlong()
        cnt = ctypes.c_longlong()
        self._chk(self.lib.csb_status(self.ctx, ctypes.byref(fl), ctypes.byref(cell),
                                      ctypes.byref(cnt), ctypes.c_void_p(self.stream)), "status")
        return int(fl.value), int(cell.value), int(cnt.value)

    def cell_ijk(self, cell):
        if cell < 0:
            return None
        if cell >= self.N:  # grid-free call with an explicit cell count
            return int(cell)
        return tuple(int(x) for x in np.unravel_index(cell, self.dims))

    def raise_for(self, flags, cell, stage="", order=("decode", "zero", "singular", "gate", "gate_decode")):
        """Raise the exception the reference raises first for these flags."""
        where = self.cell_ijk(cell)
        for kind in order:
            if kind == "decode" and flags & (F_DECODE | F_FACE_T | F_RES_NONFINITE):
                what = ("non-finite residual" if flags & F_RES_NONFINITE and not flags & (F_DECODE | F_FACE_T)
                        else "non-positive temperature at a face state" if flags & F_FACE_T and not flags & F_DECODE
                        else "non-physical state in cons_to_prim")
                raise NonPhysicalState(f"{stage}: {what} (first cell {where})")
            if kind == "zero" and flags & F_ZERO_WAVE:
                raise ZeroWavespeed(f"{stage}: all spectral radii vanish; CFL step undefined "
                                    f"(cell {where})")
            if kind == "singular" and flags & (F_SINGULAR | F_BLOCK):
                raise SingularDiagonal(f"{stage}: implicit-operator diagonal underflowed, non-finite "
                                       f"or species block not invertible (cell {where})")
            if kind == "gate" and flags & F_GATE:
                raise NonPhysicalState(f"{stage}: consistency correction / last-species "
                                       f"reconstruction went negative (first cell {where})")
            if kind == "gate_decode" and flags & F_GATE_DECODE:
                raise NonPhysicalState(f"{stage}: updated state not admissible (first cell {where})")

    def check(self, stage, order=("decode", "zero", "singular", "gate", "gate_decode")):
        flags, cell, _ = self.status()
        flags &= ~F_KSKIP
        if flags:
            self.raise_for(flags, cell, stage, order)

    # -------------------------------------------------------------- conversions
    def to_soa(self, x, nc=None):
        """Reference-layout array (numpy or torch, AoS (..., nc)) -> SoA (nc, N) on device."""
        torch = self.torch
        if isinstance(x, SoA):
            return x.t
        if isinstance(x, np.ndarray) or not hasattr(x, "data_ptr"):
            x = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float)))
            if x.numel() >= (1 << 17) and not x.is_pinned():
                # pageable input: through a page-locked bounce buffer (host copy +
                # DMA, measured 1 GB: 0.05 s against 0.10 s for the pageable copy)
                try:
                    pin = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
                    pin.copy_(x)
                    x = pin
                except RuntimeError:
                    pass
        x = x.to(device=self.device, dtype=torch.float64).contiguous()
        nc = x.shape[-1] if nc is None else nc
        n = x.numel() // nc
        out = self.empty(nc, n)
        self._chk(self.lib.csb_transpose(n, nc, x.data_ptr(), out.data_ptr(), 1,
                                         ctypes.c_void_p(self.stream)), "transpose")
        return out

    def to_host(self, t):
        """Device tensor -> numpy array.  Large results land in page-locked
        memory from torch's caching host allocator (one DMA at PCIe rate, no
        first-touch page faults; measured 1 GB: 0.02 s against 0.49 s for
        ``.cpu()``), so an array handed back to the next call also uploads at
        DMA rate.  The array owns its buffer like any other ndarray."""
        torch = self.torch
        if t.numel() * t.element_size() >= (1 << 20):
            try:
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                return h.numpy()
            except RuntimeError:  # page-locked memory exhausted: pageable copy
                pass
        return t.detach().to("cpu").numpy()

    def from_soa(self, t, like, shape):
        """SoA (nc, N) device tensor -> AoS of `shape`, numpy if `like` is numpy."""
        torch = self.torch
        nc, n = t.shape
        aos = self.empty(n, nc)
        self._chk(self.lib.csb_transpose(n, nc, t.data_ptr(), aos.data_ptr(), 0,
                                         ctypes.c_void_p(self.stream)), "transpose")
        aos = aos.reshape(shape)
        if is_torch(like):
            return aos.to(like.device)
        return self.to_host(aos)

    def from_soa_into(self, t, host):
        """SoA (nc, N) device tensor -> caller-owned AoS host tensor (N, nc)."""
        nc, n = t.shape
        aos = self.empty(n, nc)
        self._chk(self.lib.csb_transpose(n, nc, t.data_ptr(), aos.data_ptr(), 0,
                                         ctypes.c_void_p(self.stream)), "transpose")
        host.copy_(aos)
        return host

    def cells_out(self, t, like):
        """(N,) device tensor -> (ni, nj, nk) array in the caller's flavour."""
        t = t.reshape(self.dims)
        if is_torch(like):
            return t.to(like.device)
        return self.to_host(t)


class _UnitGrid:
    """1 x 1 x 1 unit box: the grid of grid-free engines (element-wise calls)."""

    dims = (1, 1, 1)

    def __init__(self, device):
        torch = torch_mod()
        f = dict(dtype=torch.float64, device=device)
        self._S = []
        for d in range(3):  # two unit faces per direction, normal along axis d
            S = torch.zeros((3, 2), **f)
            S[d] = 1.0
            self._S.append(S)
        self._vol = torch.ones(1, **f)

    def device_metrics(self, device):
        return self._S, self._vol


_UNIT = {}


def _unit_grid(device):
    g = _UNIT.get(str(device))
    if g is None:
        g = _UNIT[str(device)] = _UnitGrid(device)
    return g


class SoA:
    """A field already resident on the device in the library layout (nc, N)."""

    def __init__(self, t, dims):
        self.t = t
        self.dims = tuple(dims)


def is_torch(x):
    return hasattr(x, "data_ptr") and hasattr(x, "device") and not isinstance(x, np.ndarray)


_ENGINES = {}


class _NoGrid:
    pass


_NOGRID = _NoGrid()


_NS_MODELS = {}


def engine_for_ns(ns):
    """Grid-free engine for element-wise calls that only need the component
    count (norms, dual-time rhs): a cloned ns-species mixture."""
    m = _NS_MODELS.get(ns)
    if m is None:
        from .configs import cloned_mixture
        m = _NS_MODELS[ns] = cloned_mixture(ns)
    return get_engine(None, m)


def get_engine(grid, model, device=None):
    """Cached Engine for (grid, model); grid=None gives a grid-free engine."""
    gkey = _NOGRID if grid is None else grid
    key = (id(gkey), id(model), str(device))
    hit = _ENGINES.get(key)
    if hit is not None:
        gref, mref, eng = hit
        if gref() is gkey and mref() is model:
            return eng
    eng = Engine(grid, model, device)
    _ENGINES[key] = (weakref.ref(gkey), weakref.ref(model), eng)
    if len(_ENGINES) > 16:
        for k in list(_ENGINES)[:-16]:
            _ENGINES.pop(k, None)
    return eng
