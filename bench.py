#!/usr/bin/env python
"""Benchmark: implicit cell-iterations/s of the component-split (CS1) implicit
pseudo-time iteration on one B200 (BASELINE.json metric).

Headline workload (default ``--config 4``): BASELINE config 4, the largest
single-GPU configuration -- a 4096 x 2048 curvilinear O-grid around a unit
cylinder (stretch 1.02, wall spacing 1e-5 m), 11-species air, freestream
start (1e-3 kg/m^3, 6000 m/s, 300 K), CFL ramp 1 -> 1000.  The march is run
for ``PREP_ITERS`` accepted iterations (untimed) so the timed state carries a
developed wall layer; then one step = one full CS1 implicit iteration on that
state: residual R + grouped norms, local time step, CS operator assembly,
forward + backward LU-SGS sweeps, CS1 closure + admissibility gate.
Inputs are resident in HBM (1.07 GB of state per step, far larger than L2;
L2 is additionally flushed with a 512 MiB write before every timed step).
Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config C]

N > 1 (torchrun): independent replicas, one per GPU (the LU-SGS sweep has a
serial dependency chain; the path does not shard).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "implicit cell-iterations/s (split vs coupled) at 1 B200; % HBM roofline"
UNIT = "cell-iterations/s"
PREP_ITERS = 20          # untimed march iterations before the timed state (config 4)
CPU_SAMPLE_DIMS = {4: (256, 128, 1), 2: (128, 128, 1), 3: (128, 128, 1), 1: (128, 128, 1),
                   0: (64, 64, 1)}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--scheme", default="CS1", choices=["CS1", "CS2", "CI"])
    p.add_argument("--no-extras", action="store_true", help="skip coupled/e2e/cpu legs")
    p.add_argument("--no-scan", action="store_true", help="skip the config-2/3 scans, march, block LU")
    p.add_argument("--only", default="", help="comma list of extras to run (default: all)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_spec(cfgnum):
    from paper_2403_03440_b200 import configs as C
    if cfgnum == 0:
        return C.config0(seed=0), "config0: 64x64 box, air5 thermo, frozen chemistry, CFL 10"
    if cfgnum == 1:
        return C.config1(seed=1), "config1: 512x512 box (dx=dy=1e-3 m), air5 thermo, frozen chemistry, CFL 50"
    if cfgnum == 3:
        return C.config3(11, seed=3), "config3 ns=11: 1024x1024 box, 11-species, frozen, CFL 10"
    if cfgnum == 4:
        return C.config4(), ("config4: 4096x2048 cylinder O-grid (stretch 1.02, wall 1e-5 m), 11-species "
                             "air, freestream 1e-3 kg/m^3 / 6000 m/s / 300 K, CFL ramp 1->1000 (x2 per 45 "
                             f"it), frozen chemistry; state after {PREP_ITERS} accepted march iterations")
    raise SystemExit(f"config {cfgnum} not benchmarked")


def algorithmic_bytes(nv):
    """Canonical accounting: doubles per cell per kernel pass."""
    return {"rhs": 2 * nv + 7, "assemble": nv + 16, "sweeps": 2 * (3 * nv + 12),
            "total": 9 * nv + 47}


def march_case(spec, scheme="CS1", iters=500):
    """The drop-in ``Case`` of a config's steady march (driver.py:38-75)."""
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.driver import Case
    grid, model, bcs, mech = C.build_case(spec)
    ramp = spec.extra.get("cfl_ramp")
    return Case(grid=grid, model=model, bcs=bcs, freestream=C.freestream_of(spec, model), mech=mech,
                scheme=scheme, cfl=spec.cfl,
                cfl_ramp=(float(ramp[0]), float(ramp[1]), int(ramp[2])) if ramp else None,
                max_iters=iters, residual_drop_orders=np.inf, stop_on_absolute_floor=False)


# ---------------------------------------------------------------- clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- our arm
class Runner:
    def __init__(self, spec, scheme, q=None, cfl=None):
        import torch
        from paper_2403_03440_b200 import configs as C
        from paper_2403_03440_b200.device import SCHEMES, get_engine
        self.torch = torch
        grid, model, bcs, mech = C.build_case(spec)
        self.case_objs = (grid, model, bcs, mech)
        self.eng = eng = get_engine(grid, model)
        eng.set_bcs(bcs)
        eng.set_mechanism(mech)
        if scheme == "CI" and eng.chem_on():
            eng.ensure_workspace(True)
        self.spec = spec
        self.cfl = float(spec.cfl if cfl is None else cfl)
        self.scheme = SCHEMES[scheme]
        self.q = (q if q is not None else eng.to_soa(spec.q, eng.nv)).clone()
        self.qn = eng.empty(eng.nv, eng.N)
        self.R = eng.empty(eng.nv, eng.N)
        self.norms = eng.empty(4)
        self.lib = eng.lib
        self.stream = ctypes.c_void_p(eng.stream)
        torch.cuda.synchronize()

    def step(self, q=None, qn=None, scheme=None, norms=None, stream=None):
        e = self.eng
        st = stream if stream is not None else self.torch.cuda.current_stream().cuda_stream
        rc = self.lib.csb_iteration(e.ctx, (q if q is not None else self.q).data_ptr(), self.cfl,
                                    self.scheme if scheme is None else scheme, 0, 0,
                                    (qn if qn is not None else self.qn).data_ptr(),
                                    self.R.data_ptr(),
                                    (norms if norms is not None else self.norms).data_ptr(),
                                    ctypes.c_void_p(st))
        if rc:
            raise RuntimeError(self.lib.csb_last_error(e.ctx))

    def stages(self, reps=3, scheme=None):
        """Per-stage device time (ms) of the production path (2-D wavefront),
        instrumented pass outside the timed region."""
        torch, e, lib, st = self.torch, self.eng, self.lib, self.stream
        names = ["rhs", "norms", "srcjac", "records", "sweep_fwd", "sweep_bwd", "epilogue"]
        acc = {n: 0.0 for n in names}
        ms5 = (ctypes.c_float * 5)()
        for _ in range(reps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            lib.csb_residual(e.ctx, self.q.data_ptr(), self.R.data_ptr(), None, 0, st)
            ev[1].record()
            lib.csb_residual_norms(e.ctx, e.N, self.R.data_ptr(), self.norms.data_ptr(), st)
            ev[2].record()
            torch.cuda.synchronize()
            acc["rhs"] += ev[0].elapsed_time(ev[1])
            acc["norms"] += ev[1].elapsed_time(ev[2])
            rc = lib.csb_profile_step(e.ctx, self.q.data_ptr(), self.R.data_ptr(), self.cfl,
                                      self.scheme if scheme is None else scheme,
                                      self.qn.data_ptr(), ms5, st)
            if rc:
                raise RuntimeError(lib.csb_last_error(e.ctx))
            for k, n in enumerate(names[2:]):
                acc[n] += ms5[k]
        e.status()
        out = {n: acc[n] / reps for n in names}
        out["sweeps"] = out["sweep_fwd"] + out["sweep_bwd"]
        out["assemble"] = out["srcjac"] + out["records"]
        return out


def flush_buffer(torch):
    return torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed_steps(run, K, W, flush, scheme=None):
    """K iterations, each bracketed by CUDA events on the launching stream,
    L2 flushed before each (outside the bracket).  Returns (total ms, launches)."""
    torch = run.torch
    for _ in range(W):
        flush.zero_()
        run.step(scheme=scheme)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    l0 = run.lib.csb_launch_count()
    for a, b in evs:
        flush.zero_()
        a.record()
        run.step(scheme=scheme)
        b.record()
    torch.cuda.synchronize()
    launches = run.lib.csb_launch_count() - l0
    ms = [a.elapsed_time(b) for a, b in evs]
    return float(sum(ms)), launches


def e2e_serial(run, K, W):
    """End to end through the C ABI with HOST buffers, the way a march uses it:
    every iteration copies the state (reference layout (ni, nj, nk, nv), pinned)
    host->device, transposes it to the library layout, runs the iteration,
    transposes Q^{m+1} back and copies it and the residual norms device->host,
    all on one stream with nothing overlapped (iteration k+1 of a march needs
    Q^{m+1} of iteration k).  Returns (ms total, h2d bytes/step, d2h bytes/step)."""
    torch, e, lib = run.torch, run.eng, run.lib
    nv, N = e.nv, e.N
    host_q = torch.empty((N, nv), dtype=torch.float64).pin_memory()
    e.from_soa_into(run.q, host_q)
    host_out = torch.empty((N, nv), dtype=torch.float64).pin_memory()
    host_norms = torch.empty(4, dtype=torch.float64).pin_memory()
    dev_aos = e.empty(N, nv)
    q_soa = e.empty(nv, N)
    s = torch.cuda.current_stream()
    st = ctypes.c_void_p(s.cuda_stream)

    def one():
        dev_aos.copy_(host_q, non_blocking=True)
        lib.csb_transpose(N, nv, dev_aos.data_ptr(), q_soa.data_ptr(), 1, st)
        run.step(q=q_soa, qn=run.qn)
        lib.csb_transpose(N, nv, run.qn.data_ptr(), dev_aos.data_ptr(), 0, st)
        host_out.copy_(dev_aos, non_blocking=True)
        host_norms.copy_(run.norms, non_blocking=True)

    for _ in range(W):
        one()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        one()
    z.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(z), N * nv * 8, N * nv * 8 + 4 * 8


def e2e_pipelined(run, K, W):
    """Throughput view of the same C-ABI call over INDEPENDENT states (e.g. a
    batch of cases): the H2D of step k+1 and the D2H of step k-1 overlap the
    compute of step k on copy streams.  Not what one march can do (see
    e2e_serial); reported beside it."""
    torch, e, lib = run.torch, run.eng, run.lib
    nv, N = e.nv, e.N
    host_q = torch.empty((N, nv), dtype=torch.float64).pin_memory()
    e.from_soa_into(run.q, host_q)
    host_out = [torch.empty((N, nv), dtype=torch.float64).pin_memory() for _ in range(2)]
    host_norms = [torch.empty(4, dtype=torch.float64).pin_memory() for _ in range(2)]
    dev_aos = [e.empty(N, nv) for _ in range(2)]
    q_soa = [e.empty(nv, N) for _ in range(2)]
    qn = [e.empty(nv, N) for _ in range(2)]
    norms = [e.empty(4) for _ in range(2)]
    out_aos = [e.empty(N, nv) for _ in range(2)]
    s_comp = torch.cuda.current_stream()
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_h2d = [torch.cuda.Event() for _ in range(2)]
    ev_in_free = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]
    st = ctypes.c_void_p(s_comp.cuda_stream)
    issued = [False, False]

    def one(k):
        b = k & 1
        with torch.cuda.stream(s_h2d):
            if issued[b]:
                s_h2d.wait_event(ev_in_free[b])
            dev_aos[b].copy_(host_q, non_blocking=True)
            ev_h2d[b].record(s_h2d)
        s_comp.wait_event(ev_h2d[b])
        if issued[b]:
            s_comp.wait_event(ev_d2h[b])
        lib.csb_transpose(N, nv, dev_aos[b].data_ptr(), q_soa[b].data_ptr(), 1, st)
        ev_in_free[b].record(s_comp)
        run.step(q=q_soa[b], qn=qn[b], norms=norms[b])
        lib.csb_transpose(N, nv, qn[b].data_ptr(), out_aos[b].data_ptr(), 0, st)
        ev_comp[b].record(s_comp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_comp[b])
            host_out[b].copy_(out_aos[b], non_blocking=True)
            host_norms[b].copy_(norms[b], non_blocking=True)
            ev_d2h[b].record(s_d2h)
        issued[b] = True

    for k in range(W):
        one(k)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_comp)
    for k in range(K):
        one(W + k)
    for b in range(2):
        s_comp.wait_event(ev_d2h[b])
    z.record(s_comp)
    torch.cuda.synchronize()
    return a.elapsed_time(z)


def e2e_python_api(run, case, K=2):
    """The drop-in Python call a csflow user makes per iteration
    (reference driver.py:279, 257): ``assemble_residual(q, ...)`` then
    ``_implicit_step(case, q, R, cfl)`` with numpy AoS arrays in and out
    (wall clock, host conversions included)."""
    from paper_2403_03440_b200 import driver, spatial
    torch, e = run.torch, run.eng
    q_np = e.from_soa(run.q, np.empty(0), tuple(e.dims) + (e.nv,))
    grid, model, bcs, mech = run.case_objs
    R = spatial.assemble_residual(q_np, grid, bcs, mech, model)
    driver._implicit_step(case, q_np, R, run.cfl)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        R = spatial.assemble_residual(q_np, grid, bcs, mech, model)
        qn, _ = driver._implicit_step(case, q_np, R, run.cfl)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    return {"value": e.N / dt, "unit": UNIT, "ms_per_step": dt * 1e3, "steps": K,
            "call": "spatial.assemble_residual + driver._implicit_step, numpy AoS in/out "
                    "(pageable input, results in page-locked memory), wall clock"}


def ncu_traffic(path=os.path.join(ROOT, "profiles", "ncu_traffic.json")):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------- CPU legs
def oracle_sample(cfgnum, scheme, dims=None):
    """The CPU oracle (the reference algorithm restated in numpy/numba) on a
    bounded sample of the workload: same config distribution, `dims` cells."""
    import oracle as O
    from paper_2403_03440_b200 import configs as C
    dims = CPU_SAMPLE_DIMS.get(cfgnum, (128, 128, 1)) if dims is None else dims
    if cfgnum == 0:
        spec = C.config0(seed=0, dims=dims)
    elif cfgnum == 3:
        spec = C.config3(11, seed=3, dims=dims)
    elif cfgnum == 4:
        spec = C.config4(dims=dims)
        spec.cfl = 1.0  # cfl_at(0) of the ramp
    elif cfgnum == 2:
        spec = C.config2(dims=dims)
    else:
        spec = C.config1(seed=1, dims=dims)
    th = O.Thermo([s.M for s in spec.species], [s.cp for s in spec.species],
                  [s.hf for s in spec.species], [s.Tref for s in spec.species],
                  [s.mu_ref for s in spec.species], [s.T_mu for s in spec.species],
                  [s.S_mu for s in spec.species], spec.Pr, spec.Sc)
    grid = O.Grid(spec.nodes)
    bcs = {}
    for n, b in spec.bcs.items():
        fsv = None
        if b.fs is not None:
            rho, u, T, Y = b.fs
            fsv = O.freestream_vector(rho, u, T, Y, th)
        bcs[n] = O.BC(b.kind, Tw=b.T_wall, axis=b.axis, fs=fsv)

    def one():
        R = O.residual(spec.q, grid, bcs, None, th)
        O.norms(R)
        O.implicit_step(spec.q, R, grid, None, th, scheme, spec.cfl, want_star=False)

    return spec, one


def cpu_baseline(cfgnum, scheme, reps=5):
    spec, one = oracle_sample(cfgnum, scheme)
    _, warm = oracle_sample(cfgnum, scheme, dims=(8, 8, 1))
    warm()  # numba JIT
    one()
    t0 = time.perf_counter()
    for _ in range(reps):
        one()
    dt = (time.perf_counter() - t0) / reps
    n = spec.ncells
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle (numpy + numba sweeps, the reference algorithm restated) full "
                      f"{scheme} iteration (residual + norms + implicit step) on a "
                      f"{spec.dims[0]}x{spec.dims[1]} sample of the same config distribution, "
                      f"mean of {reps} after warm-up ({dt * reps:.1f} s); single-threaded like "
                      f"the reference (host cpu_count={os.cpu_count()})"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec_full, desc = workload_spec(args.config)
    spec, one = oracle_sample(args.config, args.scheme)
    _, warm = oracle_sample(args.config, args.scheme, dims=(8, 8, 1))
    warm()
    for _ in range(max(args.warmup, 1)):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = time.perf_counter() - t0
    n = spec.ncells
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc + f", {args.scheme} full implicit iteration", "scheme": args.scheme,
                   "sample_cells": n, "sample_grid": "x".join(map(str, spec.dims))},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"each step = one full {args.scheme} iteration (residual + norms + "
                                   f"implicit step) of the CPU oracle on a "
                                   f"{spec.dims[0]}x{spec.dims[1]} sample of the workload's "
                                   f"distribution (bounded; the reference path is serial: numba "
                                   f"sweeps, single-threaded numpy)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- config 3 scans
def species_scan(flush, nss=(5, 11, 20, 40), dims=(1024, 1024, 1), K=3, W=2):
    """Config 3 (BASELINE.json): split (CS1) vs coupled (CI) implicit
    iterations per ns on a 1024^2 box, frozen chemistry, synthetic species
    and states from seed.  Same per-step protocol as the headline (L2 flushed,
    CUDA events)."""
    import torch
    from paper_2403_03440_b200 import configs as C
    out = []
    for ns in nss:
        spec = C.config3(ns, dims=dims)
        run = Runner(spec, "CS1")
        cs_ms, _ = timed_steps(run, K, W, flush)
        ci_ms, _ = timed_steps(run, K, W, flush, scheme=0)
        run.eng.status()
        N = run.eng.N
        out.append({"ns": ns, "split_CS1": N * K / (cs_ms * 1e-3),
                    "coupled_CI": N * K / (ci_ms * 1e-3),
                    "coupled_path": "wavefront (register chain)" if ns <= 16
                    else "wavefront (smem-resident chain, ns > 16)"})
        del run
        torch.cuda.empty_cache()
    return {"unit": UNIT, "grid": "x".join(map(str, dims)), "chemistry": "frozen",
            "steps": K, "results": out}


def chemistry_scan(flush, nss=(5, 11, 20, 40), dims=(1024, 1024, 1), K=2, W=1):
    """Config 3 with chemistry: synthetic mechanisms (2 ns reversible
    reactions, BASELINE config-3 recipe), CS1 vs CI per ns on the 1024^2 box.
    The iteration includes the FD source Jacobian (reference
    chemistry.py:76-104); CI with chemistry adds the species block inverse
    inv(d I - V dOmega) per cell (implicit.py:362-368) and runs on the
    wavefront up to 16 species (generic hyperplane sweeps above).  The synthetic
    mechanisms are extremely stiff: the gate flags most cells,
    which does not change the work done."""
    import torch
    from paper_2403_03440_b200 import configs as C
    out = []
    for ns in nss:
        spec = C.config3(ns, dims=dims, chemistry=True)
        run = Runner(spec, "CI")  # CI workspace (block inverse) allocated up front
        from paper_2403_03440_b200.device import SCHEMES
        cs_ms, _ = timed_steps(run, K, W, flush, scheme=SCHEMES["CS1"])
        st_cs = run.stages(reps=1, scheme=SCHEMES["CS1"])
        ci_ms, launches = timed_steps(run, K, W, flush, scheme=SCHEMES["CI"])
        run.eng.status()
        N = run.eng.N
        out.append({"ns": ns, "reactions": 2 * ns, "split_CS1": N * K / (cs_ms * 1e-3),
                    "coupled_CI": N * K / (ci_ms * 1e-3),
                    "split_ms": cs_ms / K, "coupled_ms": ci_ms / K,
                    "split_srcjac_ms": st_cs["srcjac"],
                    "coupled_path": ("wavefront (register CI chain, ns x ns block inverses in the "
                                     "records)" if ns <= 16 else
                                     "generic hyperplane sweeps (graph-replayed) + block inverse"),
                    "coupled_launches_per_step": launches / K})
        del run
        torch.cuda.empty_cache()
    return {"unit": UNIT, "grid": "x".join(map(str, dims)), "chemistry": "synthetic mechanisms",
            "steps": K, "results": out}


def config2_run(flush, iters=10, cfl_march=0.1):
    """Config 2: 1024^2 O-grid, 11 species, smoothed random fields, 10 CS1
    iterations at CFL 100.  SURVEY G11: the reference driver raises Diverged
    on the first step here (admissibility fails next to the 300 K wall for
    any CFL above ~0.1), so two measurements stand in for it:
    (i) one iteration at CFL 100 from the initial state, timed per step with
        the gate evaluated and counted, not acted on (function level);
    (ii) the 10-iteration march through steady_solve (device march) at the
        largest admissible CFL, 0.1."""
    import torch
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.driver import Case, steady_solve
    spec = C.config2()
    run = Runner(spec, "CS1")
    K = 3
    ms, _ = timed_steps(run, K, 1, flush)
    fl, cell, cnt = run.eng.status()
    N = run.eng.N
    grid, model, bcs, mech = run.case_objs
    case = Case(grid=grid, model=model, bcs=bcs, freestream=C.freestream_of(spec, model),
                mech=mech, scheme="CS1", cfl=cfl_march, max_iters=iters,
                residual_drop_orders=np.inf, stop_on_absolute_floor=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    q, hist = steady_solve(case, spec.q, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"grid": "1024x1024", "ns": 11,
           "g11_options": "(i) one iteration at CFL 100, gate counted; (ii) 10-iteration march at "
                          f"CFL {cfl_march} (the reference's retry loop diverges at CFL 100)",
           "cfl100_ms_per_iteration": ms / K, "cfl100_cell_it_per_s": N * K / (ms * 1e-3),
           "cfl100_gate_failures_per_iteration": int(cnt) // K,
           "march_iterations": len(hist.iters), "march_retries": int(sum(hist.retries)),
           "march_wall_s": wall, "march_cell_it_per_s": N * len(hist.iters) / wall,
           "march_reason": hist.reason}
    del run
    torch.cuda.empty_cache()
    return out


def march500(iters=500):
    """Config 4's full march through the drop-in ``steady_solve``: 500
    iterations, CFL ramp 1 -> 1000 (x2 every 45), halving retries with x1.2
    recovery (driver.py:254-263, 308-313).  Sustained accepted cell-it/s =
    accepted iterations x cells / wall time (retried steps cost time but do
    not count)."""
    import torch
    from paper_2403_03440_b200 import configs as C
    from paper_2403_03440_b200.driver import steady_solve
    spec = C.config4()
    case = march_case(spec, "CS1", iters)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    q, hist = steady_solve(case, spec.q, return_device=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    N = spec.ncells
    acc = len(hist.iters)
    return {"grid": "4096x2048", "ns": 11, "iterations": acc, "retries": int(sum(hist.retries)),
            "wall_s": wall, "sustained_cell_it_per_s": N * acc / wall,
            "implicit_s": float(sum(hist.implicit_seconds)),
            "cfl_final": hist.cfl[-1] if hist.cfl else None, "reason": hist.reason,
            "res_density_first_last": [hist.res_density[0], hist.res_density[-1]],
            "res_flow_every_50": hist.res_flow[::50], "cfl_every_50": hist.cfl[::50]}


# ---------------------------------------------------------------- FP64 block LU
def fp64_peak_tflops(lib, torch):
    """Measured FP64 pipe peak (csb_fp64_peak: independent DFMA chains on
    every SM), the denominator of the block-inverse roofline."""
    scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    iters = 4000
    lib.csb_fp64_peak(50, scratch.data_ptr(), st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.csb_fp64_peak(iters, scratch.data_ptr(), st)
    b.record()
    torch.cuda.synchronize()
    flops = sms * 4 * 256 * iters * 16 * 8 * 2.0
    return flops / (a.elapsed_time(b) * 1e-3) / 1e12


def block_lu(hbm_peak, nss=(5, 11, 20, 32), N=1 << 20, reps=5):
    """Batched species block inverse inv(d I - V dOmega) of the coupled
    operator with chemistry (reference implicit.py:362-368) on N = 2^20 cells
    (config-3 cell count) per ns: achieved FP64 TFLOP/s (2 n^3 flops per
    cell, Gauss-Jordan = LAPACK getrf + getri count) against the measured
    FP64 peak, and algorithmic bytes (2 n^2 + 2 doubles per cell) against
    HBM.  ``binding`` names the larger of the two fractions (the roofline the
    kernel is closer to); ``latency_bound`` is set when both are below 50 %."""
    import torch
    from paper_2403_03440_b200 import _lib
    lib = _lib.load()
    peak = fp64_peak_tflops(lib, torch)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(7)
    out = []
    for ns in nss:
        dom = torch.randn((ns * ns, N), generator=g, device="cuda", dtype=torch.float64)
        d = torch.rand(N, generator=g, device="cuda", dtype=torch.float64) * ns + ns
        V = torch.ones(N, device="cuda", dtype=torch.float64)
        dinv = torch.empty_like(dom)
        fl = torch.zeros(16, dtype=torch.int64, device="cuda")
        lib.csb_batched_inverse(ns, N, dom.data_ptr(), d.data_ptr(), V.data_ptr(), dinv.data_ptr(),
                                fl.data_ptr(), st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            lib.csb_batched_inverse(ns, N, dom.data_ptr(), d.data_ptr(), V.data_ptr(),
                                    dinv.data_ptr(), fl.data_ptr(), st)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        tf = 2.0 * ns ** 3 * N / (ms * 1e-3) / 1e12
        gbs = (2 * ns * ns + 2) * 8.0 * N / (ms * 1e-3) / 1e9
        ff, hf = tf / peak, gbs / hbm_peak
        out.append({"ns": ns, "ms": ms, "tflops": tf, "fp64_frac": ff, "gbs": gbs,
                    "hbm_frac": hf, "binding": "fp64" if ff >= hf else "hbm",
                    "latency_bound": bool(max(ff, hf) < 0.5)})
        del dom, dinv
    return {"cells": N, "fp64_peak_tflops": peak,
            "fp64_peak_source": "measured live (csb_fp64_peak DFMA chains, all SMs)",
            "flops_per_cell": "2 ns^3", "bytes_per_cell": "(2 ns^2 + 2) x 8", "results": out}


# ---------------------------------------------------------------- replicas
def replica_aggregate(local_ms, cells_per_rank, steps, dist=None, device="cpu"):
    """Whole-job throughput of N independent replicas: the timed region's
    device time is the MAX over ranks, value = cells all ranks processed /
    that time.  Returns (value, max_ms).  Works with any torch.distributed
    backend (nccl on the GPU box, gloo in the CPU tests)."""
    import torch
    world = dist.get_world_size() if dist is not None else 1
    t = torch.tensor([float(local_ms)], device=device, dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    return world * cells_per_rank * steps / (max_ms * 1e-3), max_ms


def prepare(spec, cfgnum, scheme):
    """(Runner, case-or-None): config 4 marches PREP_ITERS accepted
    iterations from the freestream first (untimed) and times the state it
    reaches at the CFL the ramp gives next."""
    if cfgnum != 4:
        return Runner(spec, scheme), None
    from paper_2403_03440_b200.driver import steady_solve
    case = march_case(spec, scheme, PREP_ITERS)
    q, hist = steady_solve(case, spec.q, return_device=True)
    cfl = case.cfl_at(PREP_ITERS)
    run = Runner(spec, scheme, q=q.t, cfl=cfl)
    return run, case


# ---------------------------------------------------------------- main
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    only = set(x for x in args.only.split(",") if x)
    want = lambda k: not only or k in only
    spec, desc = workload_spec(args.config)
    run, case = prepare(spec, args.config, args.scheme)
    flush = flush_buffer(torch)
    # settle clocks (untimed), then sample clocks across warm-up + timed region
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        run.step()
        torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms, launches = timed_steps(run, args.steps, args.warmup, flush)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    fl, cell, gate = run.eng.status()
    N = run.eng.N
    nv = run.eng.nv
    value, total_ms = replica_aggregate(total_ms, N, args.steps, dist, device="cuda")

    extras = {}
    e2e = None
    if not args.no_extras:
        # split vs coupled at equal care: the CI operator on the same workload
        kci = max(3, args.steps // 2)
        ci_ms, _ = timed_steps(run, kci, 2, flush, scheme=0)
        extras["coupled_CI"] = {"value": N * kci / (ci_ms * 1e-3), "unit": UNIT,
                                "ms_per_step": ci_ms / kci}
        run.eng.status()
        ke = max(3, args.steps // 2)
        e2e_ms, h2d, d2h = e2e_serial(run, ke, 1)
        pip_ms = e2e_pipelined(run, ke, 1)
        e2e = {"value": world * N * ke / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_ms / ke, "mode": "serial (one march iteration: H2D, transpose, "
                                                   "iteration, transpose, D2H; nothing overlapped)",
               "pipelined": {"value": world * N * ke / (pip_ms * 1e-3), "unit": UNIT,
                             "ms_per_step": pip_ms / ke,
                             "mode": "independent states, copies overlapped with compute"}}
        if case is not None and want("python_api"):
            try:
                e2e["python_api"] = e2e_python_api(run, case)
            except Exception as exc:
                e2e["python_api"] = {"error": repr(exc)}
        run.eng.status()
    stages = run.stages()
    ab = algorithmic_bytes(nv)
    peak, peak_src = peaks()
    dom = max(("rhs", "sweeps", "assemble"), key=lambda k: stages[k])
    dom_ms = stages[dom]
    bytes_dom = N * ab[dom] * 8
    achieved = bytes_dom / (dom_ms * 1e-3) / 1e9
    traffic = None
    tr = ncu_traffic()
    if tr and tr.get("workload") == f"config{args.config}" and dom in tr.get("per_launch_bytes", {}):
        traffic = tr["per_launch_bytes"][dom]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                "algorithmic_bytes_per_cell": ab[dom] * 8, "peak_source": peak_src,
                "note": "achieved = SURVEY §8(d) algorithmic bytes of the stage / its CUDA-event time"}
    per_stage = {}
    for k in ("rhs", "assemble", "sweeps"):
        gbs = N * ab[k] * 8 / (stages[k] * 1e-3) / 1e9
        per_stage[k] = {"ms": stages[k], "gbs": gbs, "frac": gbs / peak}
    if tr and tr.get("workload") == f"config{args.config}" and "fp64" in tr and dom == "rhs":
        # the residual is FP64-issue bound, not HBM bound: its instruction
        # roofline (ncu instruction counts x this run's stage time)
        f = dict(tr["fp64"])
        f["frac_of_fp64_pipe"] = f["fp64_bound_ms"] / dom_ms
        f["frac_of_issue_bound"] = f["issue_bound_ms"] / dom_ms
        roofline["fp64"] = f
    if not args.no_extras and not args.no_scan:
        for key, fn in (("species_scan", lambda: species_scan(flush)),
                        ("chemistry_scan", lambda: chemistry_scan(flush)),
                        ("config2", lambda: config2_run(flush)),
                        ("march500", lambda: march500()),
                        ("block_lu", lambda: block_lu(peak))):
            if not want(key):
                continue
            try:
                extras[key] = fn()
            except Exception as exc:  # extras must not kill the headline line
                extras[key] = {"error": repr(exc)}
            torch.cuda.empty_cache()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc + f", {args.scheme} full implicit iteration per step",
                   "grid": "x".join(map(str, spec.dims)), "ns": spec.ns, "scheme": args.scheme,
                   "cfl": run.cfl, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs (1 GB state) larger than L2, and L2 flushed (512 MiB device "
                         "write) before every timed step",
                   "inputs": "resident in HBM (value); host pinned buffers (e2e)"},
        "roofline": roofline,
        "stages_ms": stages,
        "stage_roofline": per_stage,
        "iteration_roofline_frac": (N * ab["total"] * 8 / (total_ms / args.steps * 1e-3) / 1e9) / peak,
        "gate_failures": gate,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk,
    }
    if e2e is not None:
        line["e2e"] = e2e
    line.update(extras)
    if rank == 0 and not args.no_extras:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, args.scheme)
        except Exception as exc:  # the CPU leg must not kill the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
