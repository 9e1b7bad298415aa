#!/usr/bin/env python
"""Benchmark: value + gradient + HVP summand evaluations of BASELINE.json
configs[1] (L=8 spinful Fermi-Hubbard, 16 qubits, 5 layers / 36 slots, Haar
gates seed 1, target exp(-iHt) with J=1, U=4, t=0.25).

A *summand* is one basis state |j> of the basis sum: its value phi0 . C|j>,
its gradient holes (reference _gradient_chunk, objective.py:322-337) and its
HVP holes along the seeded tangent direction (reference _hvp_chunk,
objective.py:432-482).  The metric is summands per second; the full-sum
figure (one evaluation = all 2^16 summands) is derived beside it
(``full_sum_evals_per_s``).

* B200 arm (default): one step = one full-sum evaluation (65536 summands),
  fused into one reversible 3-sweep pass per summand by the engine.  With N
  GPUs (torchrun, or self-launched by ``--gpus N``) the fixed basis sum is
  sharded over ranks in contiguous chunks (strong scaling); the only
  collective is the all-gather of per-chunk records.
* ``--impl reference``: the reference algorithm's CPU implementation (the C
  port in oracle/, restating the reference drivers) on every host thread;
  one step = a bounded 64-summand sample of the same workload.  The circuit
  and direction are read from tests/golden/c2_slice.npz, which the unmodified
  reference wrote; nothing of the product package is imported.

In both arms ``value`` excludes target generation (phi0 precomputed: cached
HBM columns on the GPU, Lanczos columns on the host); the target-inclusive
variants are reported beside it (``e2e`` on the GPU, ``with_target`` on the
host).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gradient+HVP evals/sec at 16-site Hubbard; gate-apply HBM GB/s vs peak"
UNIT = "gradient+HVP summand-evals/s"
L_SITES, LAYERS, SEED, T_EVOL = 8, 5, 1, 0.25
K_QUBITS = 2 * L_SITES
TOTAL = 1 << K_QUBITS
REF_SAMPLE = 64  # summands per reference-arm step
# identical in both arms (the driver compares them)
CONFIG = {
    "workload": "c2 (BASELINE configs[1]): spinful Fermi-Hubbard L=8 open, 16 qubits, J=1 U=4 t=0.25; circuit 5 "
                "layers = 36 slots / 5 logical Haar gates (seed 1); per summand |j>: value + gradient + one HVP "
                "along the seeded tangent direction",
    "full_sum_summands": TOTAL,
    "targets": "phi0 = conj(exp(-iHt)|j>) precomputed outside the timed region (target-inclusive variant reported "
               "separately)",
    "parallelism": "basis-sum data parallel",
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload():
    import paper_2506_23775_b200 as gf

    spec, circ, rng = gf.spinful_layer_circuit(L_SITES, LAYERS, False, seed=SEED)
    X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))
         for g in circ.logical_gates]
    return gf, spec, circ, X


class Clocks:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# process group
# ---------------------------------------------------------------------------


def _self_launch(args) -> int:
    """``--gpus N`` outside torchrun: start N ranks with torch.distributed.run
    on 127.0.0.1 and return their exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _dist(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    ngpu = torch.cuda.device_count()
    # --backend gloo on a one-GPU box: ranks share cuda:0 (CPU test of the multi-rank path only)
    dev = local if args.backend == "nccl" else local % max(ngpu, 1)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    return rank, world, dev, (dist if world > 1 else None)


def _reduce_over_ranks(x, dist, op):
    import torch

    if dist is None:
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def _max_over_ranks(x, dist):
    return x if dist is None else _reduce_over_ranks(x, dist, dist.ReduceOp.MAX)


def _sum_over_ranks(x, dist):
    return x if dist is None else _reduce_over_ranks(x, dist, dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------


def measure_fp64_peaks(gf):
    """FP64 tensor (DMMA m8n8k4) and FMA peaks of this GPU, measured in-run."""
    import torch

    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    out = {}
    st = gf._lib.stream_ptr()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for which, key in ((0, "dmma_tflops"), (1, "dfma_tflops")):
        fl = np.zeros(1)
        gf._lib.check(gf._lib.lib.gf_peak_fp64(which, 148 * 4, 64, sink.data_ptr(), fl.ctypes.data, st))
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            e0.record(stream)
            gf._lib.check(gf._lib.lib.gf_peak_fp64(which, 148 * 4, 2048, sink.data_ptr(), fl.ctypes.data, st))
            e1.record(stream)
            torch.cuda.synchronize()
            best = max(best, fl[0] / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        out[key] = round(best, 2)
    return out


def gate_apply_sweep(gf, peak):
    """Standalone K1 bandwidth sweep on one 2^31-amplitude complex128 vector
    (the c5 compressed 31-qubit space, 32 GiB): 2q adjacent (t, t+1), 2q long
    range (t, t+15 mod 31), the generic 1q gate on every qubit and the
    parity-controlled 1q gate of the implicit qubit; in place, 32 B per
    amplitude per application."""
    import torch

    K = 31
    N = 1 << K
    try:
        x = torch.empty(N, dtype=torch.complex128, device="cuda")
    except RuntimeError:
        K, N = 30, 1 << 30
        x = torch.empty(N, dtype=torch.complex128, device="cuda")
    x.real.normal_()
    x.imag.normal_()
    rng = np.random.default_rng(0)
    st = gf._lib.stream_ptr()
    stream = torch.cuda.current_stream()
    cases = [("adj", t, t + 1) for t in range(K - 1)] + [("long", t, (t + 15) % K) for t in range(K)]
    cases += [("1q", a, None) for a in range(K)]
    cases += [("c1q", a, None) for a in range(K)]
    results = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for kind, a, b in cases:
        if kind == "c1q":
            g = gf.manifold.parity_join(gf.manifold.random_unitary(2, rng), gf.manifold.random_unitary(2, rng))
        elif kind == "1q":
            g = gf.manifold.random_unitary(2, rng)
        else:
            g = gf.manifold.random_unitary(4, rng)
        g = np.ascontiguousarray(g)

        def launch():
            if kind == "c1q":
                gf._lib.check(gf._lib.lib.gf_apply_gate_sector_c1q(x.data_ptr(), x.data_ptr(), K + 1, a, 0,
                                                                   g.ctypes.data, 1, st))
            elif kind == "1q":
                gf._lib.check(gf._lib.lib.gf_apply_gate_1q(x.data_ptr(), x.data_ptr(), K, a, g.ctypes.data, 1, st))
            else:
                gf._lib.check(gf._lib.lib.gf_apply_gate(x.data_ptr(), x.data_ptr(), K, a, b, g.ctypes.data, 0, 1,
                                                        st))

        launch()
        torch.cuda.synchronize()
        e0.record(stream)
        reps = 3
        for _ in range(reps):
            launch()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = 32.0 * N / (ms * 1e-3) / 1e9
        results.append((kind, a, b, ms, gbs))
    del x
    torch.cuda.empty_cache()
    g_all = np.array([r[4] for r in results])
    worst = min(results, key=lambda r: r[4])
    return {
        "vector_amplitudes": N,
        "bytes_per_application": 32 * N,
        "launches": len(results) * 4,
        "gbs_median": round(float(np.median(g_all)), 1),
        "gbs_min": round(float(g_all.min()), 1),
        "gbs_max": round(float(g_all.max()), 1),
        "frac_of_measured_peak_median": round(float(np.median(g_all)) / peak, 4),
        "frac_of_8TBs_nominal_median": round(float(np.median(g_all)) / 8000.0, 4),
        "worst_case": f"{worst[0]} ({worst[1]},{worst[2]}) {worst[4]:.0f} GB/s",
        "per_case_gbs": {f"{r[0]}:{r[1]}-{r[2]}": round(r[4], 1) for r in results},
    }


def cpu_gate_apply(k=24):
    """The CPU port of the reference gate kernel (oracle/gf_oracle.c restating
    kernels.py:132-205, one thread as numba runs each call) on a 2^k vector:
    GB/s at 32 B per amplitude for an adjacent, a strided and a long-range
    target pair (cli.py:424-441 style)."""
    from oracle import gf_oracle as O

    rng = np.random.default_rng(3)
    psi = (rng.standard_normal(1 << k) + 1j * rng.standard_normal(1 << k)).astype(np.complex128)
    g = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))[0]
    out = {}
    for a, b in ((k - 2, k - 1), (0, 1), (3, k - 4)):
        O.apply_gate(psi, g, (a, b))  # warm
        t0 = time.perf_counter()
        O.apply_gate(psi, g, (a, b))
        dt = time.perf_counter() - t0
        out[f"({a},{b})"] = round(32.0 * (1 << k) / dt / 1e9, 2)
    return {"vector_amplitudes": 1 << k, "threads": 1, "gbs": out}


def port_grad_hvp(plan, X, js, phi_rows, workers):
    """Oracle port (oracle/gf_oracle.c, restating the reference drivers
    _gradient_chunk + _hvp_chunk, objective.py:322-337, 432-482) on the host:
    gradient + HVP of every summand of js, spread over `workers` threads (the
    reference's parallel_reduce over its ThreadPoolExecutor).  Returns
    (seconds, value sum)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import gf_oracle as O

    parts = [p for p in np.array_split(np.arange(len(js)), workers) if len(p)]

    def work(sel):
        jj = js[sel]
        P = phi_rows[sel]
        fn = lambda q: P[np.searchsorted(jj, q)]
        v, _, _ = O.gradient_sum(plan, jj, fn)
        O.hvp_sum(plan, X, jj, fn)
        return v

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=workers) as ex:
        v = sum(ex.map(work, parts))
    return time.perf_counter() - t0, v


def lanczos_rows(js, workers):
    """phi0 rows of js from the oracle's restatement of the reference
    KrylovOracle (models.py:322-384); returns (rows, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import gf_oracle as O

    terms, _ = O.spinful_terms(L_SITES, 1.0, 4.0, False)
    fn = O.lanczos_phi0(K_QUBITS, terms, T_EVOL)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=workers) as ex:
        rows = list(ex.map(lambda j: fn(np.array([j]))[0], js))
    return np.ascontiguousarray(np.stack(rows)), time.perf_counter() - t0


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port; the reference itself is numba and cannot travel) on all host
    threads.  Each step evaluates gradient + HVP of a fixed seeded sample of
    REF_SAMPLE c2 summands; ms_per_step is the measured wall time of one step.
    The circuit, gates and direction come from the reference-written fixture
    tests/golden/c2_slice.npz (identical to the B200 arm's recipe, checked by
    tests/test_host_logic.py)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import gf_oracle as O

    d = np.load(os.path.join(ROOT, "tests", "golden", "c2_slice.npz"))
    plan = O.Plan(int(d["k"]), d["targets"], d["logical"], d["gates"])
    X = list(d["direction"])
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    js = np.sort(rng.choice(TOTAL, size=REF_SAMPLE, replace=False)).astype(np.int64)
    rows, lanczos_s = lanczos_rows(js, cores)  # setup: targets are outside `value` in both arms
    times = []
    for step in range(args.warmup + args.steps):
        dt, _ = port_grad_hvp(plan, X, js, rows, cores)
        if step >= args.warmup:
            times.append(dt)
    tot = float(np.sum(times))
    v = REF_SAMPLE * len(times) / tot
    target_rate = REF_SAMPLE / lanczos_s
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic: BASELINE configs[1] circuit and direction from tests/golden/c2_slice.npz (written by the "
                "unmodified reference); targets from the Lanczos restatement of the reference KrylovOracle",
        "config": CONFIG,
        "step": f"gradient + HVP of a fixed seeded sample of {REF_SAMPLE} summands (reference _gradient_chunk + "
                f"_hvp_chunk restated in oracle/gf_oracle.c) on {cores} host threads",
        "full_sum_evals_per_s": v / TOTAL,
        "with_target": {"value": 1.0 / (1.0 / v + 1.0 / target_rate), "unit": UNIT,
                        "lanczos_summands_per_s": target_rate,
                        "note": "Lanczos target column per summand included (the reference _phi_block path)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{REF_SAMPLE} seeded c2 summands per step, gradient + HVP each, phi0 "
                                   f"precomputed"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# c5 secondary measurement (BASELINE configs[4], one summand)
# ---------------------------------------------------------------------------


def c5_summand(gf, peaks64):
    """One c5 summand (L=16 periodic, 32 qubits, even sector compressed to
    2^31 amplitudes, 144 slots / 9 logical, folded orbit representative):
    value + gradient + one HVP on the sector's FMA unit engine (PM_UNIT).
    Algorithmic FP64 flops per summand: per amplitude per slot 9 parity-gate
    applications at 16 flop + 3 holes at 16 flop (their 8 on-pattern entries)
    = 192 flop, exactly what the unit engine executes.  `flops_dense_holes`
    keeps the r01 / r02a count (2q holes at their full 16 entries, 32 flop)."""
    import torch

    spec, circ, rng = gf.spinful_layer_circuit(16, 9, True, seed=4, parity=True)
    X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), True)
         for g in circ.logical_gates]
    k = circ.num_qubits
    N = 1 << (k - 1)
    srng = np.random.default_rng(5)
    i0 = int(srng.integers(0, N))
    x = torch.tensor([i0], dtype=torch.int64, device="cuda")
    full, rep, size, comp = (torch.empty_like(x) for _ in range(4))
    st = gf._lib.stream_ptr()
    gf._lib.check(gf._lib.lib.gf_sector_unrank(x.data_ptr(), 1, 0, full.data_ptr(), st))
    gf._lib.check(gf._lib.lib.gf_orbit_canon(full.data_ptr(), 1, 16, rep.data_ptr(), size.data_ptr(), st))
    gf._lib.check(gf._lib.lib.gf_sector_rank(rep.data_ptr(), 1, comp.data_ptr(), st))
    basis = (comp.cpu().numpy(), size.cpu().numpy().astype(np.float64))
    orc = gf.NumberBlockOracle(spec, T_EVOL)
    cache = gf.models.CachedTargetColumns(orc, k, 0, 1, sector=0, indices=basis[0], batch=1)
    del orc
    torch.cuda.empty_cache()
    gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)  # plan + warm-up
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)
    e1.record(stream)
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    t1, t2, _ = circ.slot_arrays()
    n1q = int(np.sum((t1 == k - 1) | (t2 == k - 1)))
    n2q = circ.num_slots - n1q
    flops = float(N) * circ.num_slots * (9 * 16 + 3 * 16)
    flops_dense = float(N) * (n2q * (9 * 16 + 3 * 32) + n1q * (9 * 16 + 3 * 16))
    dmma_peak, dfma_peak = peaks64["dmma_tflops"], peaks64["dfma_tflops"]
    from paper_2506_23775_b200 import objective as obj

    shape = list(obj._PLANS.values())[-1].describe()
    lf = shape.get("live_fraction", {"forward": 1.0, "reverse": 1.0, "ascending": 1.0})
    # executed flops: the light-cone rule skips the tiles on which psi is zero
    # (per amplitude per slot: forward 16, reverse 96, ascending 80 flop)
    executed = float(N) * circ.num_slots * (16 * lf["forward"] + 96 * lf["reverse"] + 80 * lf["ascending"])
    obj._PLANS.clear()
    del cache
    torch.cuda.empty_cache()
    return {"config": "c5 (BASELINE configs[4]): L=16 periodic, 32 qubits, even sector (2^31 amplitudes), fold, "
                      "144 slots / 9 logical; one summand value + gradient + HVP",
            "summand_evals_per_s": 1.0 / s, "s_per_summand": s, "fp64_tflops": executed / s / 1e12,
            "frac_of_dfma_peak": executed / s / 1e12 / dfma_peak, "frac_of_dmma_peak": executed / s / 1e12 / dmma_peak,
            "executed_flops": executed, "live_fraction": lf,
            "algorithmic_flops": flops, "fp64_tflops_algorithmic": flops / s / 1e12,
            "flops_dense_holes": flops_dense,
            "fp64_tflops_dense_holes": flops_dense / s / 1e12,
            "frac_of_dmma_peak_dense_holes": flops_dense / s / 1e12 / dmma_peak,
            "bound": "FP64 FMA pipe + shared-memory wavefronts (two-amplitude units, DFMA with uniform-register "
                     "matrix operands); B200's DMMA and DFMA share one FP64 datapath",
            "engine": shape}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def run_b200(args):
    import torch

    rank, world, dev, dist = _dist(args)
    gf, spec, circ, X = workload()
    from paper_2506_23775_b200 import objective as obj

    peak, peak_src = _peaks()
    chunk = obj.CHUNK_STATES
    N = TOTAL
    summands = min(args.summands, TOTAL) if args.summands else TOTAL
    nchunks = (summands + chunk - 1) // chunk
    lo, hi = obj.shard_chunks(nchunks, rank, world)  # this rank's positions of the basis sum
    p0, p1 = lo * chunk, min(summands, hi * chunk)
    batch = args.batch or obj._default_batch(N, TOTAL)
    make_target = {"blocks": gf.NumberBlockOracle, "chebyshev": gf.ChebyshevOracle}[args.oracle]
    oracle = make_target(spec, T_EVOL)
    t_or = time.perf_counter()
    sel = np.arange(summands, dtype=np.int64) if args.summands else None
    cache = gf.models.CachedTargetColumns(oracle, K_QUBITS, p0, max(p1, p0), indices=sel, batch=batch)
    torch.cuda.synchronize()
    oracle_setup_s = time.perf_counter() - t_or
    kw = dict(batch=batch, distributed=(dist is not None))
    if args.summands:
        kw["basis"] = sel
    for _ in range(args.warmup):
        rep, hv = gf.gradient_and_hvp(circ, cache, X, **kw)
    torch.cuda.synchronize()
    plan = next(iter(obj._PLANS.values()))
    plan_shape = plan.describe()
    gf._lib.check(gf._lib.lib.gf_plan_set_profiling(plan.h, 1))

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(dev)
    clk.start()
    launches = 0
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        rep, hv = gf.gradient_and_hvp(circ, cache, X, **kw)
        launches += rep.engine["launches"]
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    ms_max = _max_over_ranks(ms, dist)
    launches_all = int(_sum_over_ranks(launches, dist))
    value = summands * args.steps / (ms_max * 1e-3)

    ms4 = np.zeros(4)
    l4 = np.zeros(4, dtype=np.int64)
    gf._lib.check(gf._lib.lib.gf_plan_phase_times(plan.h, ms4.ctypes.data, l4.ctypes.data))
    import ctypes as _ct
    r1_ms, r1_l, r1_v, r1_s = _ct.c_double(0), _ct.c_int64(0), _ct.c_int64(0), _ct.c_int(0)
    gf._lib.check(gf._lib.lib.gf_plan_first_reverse_pass(plan.h, _ct.byref(r1_ms), _ct.byref(r1_l), _ct.byref(r1_v),
                                                         _ct.byref(r1_s)))
    gf._lib.check(gf._lib.lib.gf_plan_set_profiling(plan.h, 0))
    n = circ.num_slots
    my_summands = (p1 - p0) * args.steps
    peaks64 = measure_fp64_peaks(gf)
    # algorithmic FP64 flops per amplitude per slot (dense 4x4 complex gate on a
    # 4-amplitude tuple = 16 complex MACs = 32 flop per amplitude; a hole
    # contraction is the same count): forward G psi = 1; reverse G^dag psi, two
    # holes, G^T chi, Z^T bra, G^T bra = 6; ascending conj(G) bra, hole, G v,
    # Z psi, G psi = 5
    mv = 32.0 * N * n * my_summands
    flops_phase = {"forward": 1 * mv, "reverse": 6 * mv, "ascending": 5 * mv}
    # light cone of the basis states: the engine skips the tiles on which
    # psi_l = G_l..G_1|j> is exactly zero (gf_plan_live_fraction); executed
    # flops = algorithmic flops (what the reference's full-vector passes do) x
    # the live fraction of the slot work
    live = plan_shape.get("live_fraction", {"forward": 1.0, "reverse": 1.0, "ascending": 1.0})
    # HBM bytes, fused pass model: every pass reads + writes each touched
    # vector once (forward psi; reverse psi, bra, chi; ascending psi, bra, v)
    vec_bytes = 32.0 * N * batch
    pass_bytes = {"forward": 1 * vec_bytes, "reverse": 3 * vec_bytes, "ascending": 3 * vec_bytes}
    phases = {}
    names = ("forward", "reverse", "ascending", "reduce")
    for i, nm in enumerate(names):
        phases[nm] = {"ms": round(float(ms4[i]), 3), "launches": int(l4[i]),
                      "share": round(float(ms4[i] / ms4.sum()), 4) if ms4.sum() else None}
        if nm in flops_phase and ms4[i] > 0:
            phases[nm]["fp64_tflops"] = round(live[nm] * flops_phase[nm] / (ms4[i] * 1e-3) / 1e12, 3)
            phases[nm]["fp64_tflops_algorithmic"] = round(flops_phase[nm] / (ms4[i] * 1e-3) / 1e12, 3)
            phases[nm]["live_fraction"] = round(live[nm], 4)
            phases[nm]["hbm_gbs_pass_model"] = round(pass_bytes[nm] * l4[i] / (ms4[i] * 1e-3) / 1e9, 1)
    dom = max(("forward", "reverse", "ascending"), key=lambda k: ms4[names.index(k)])
    achieved = phases[dom]["fp64_tflops"]
    # the dominant launch: the reverse sweep's first pass (every tile live, so
    # executed = algorithmic flops): 6 units of 32 flop per amplitude per slot
    rev1 = None
    if r1_ms.value > 0 and r1_l.value > 0:
        fl = 6 * 32.0 * N * r1_s.value * r1_v.value
        rev1 = {"kernel": "k_fused<OP_REV_GH, FIRST>: first reverse pass, %d slots, every tile live" % r1_s.value,
                "launches": int(r1_l.value), "ms_per_launch": round(r1_ms.value / r1_l.value, 4),
                "share_of_step": round(r1_ms.value / ms4.sum(), 4) if ms4.sum() else None,
                "fp64_tflops": round(fl / (r1_ms.value * 1e-3) / 1e12, 3)}
        if dom == "reverse":
            achieved = rev1["fp64_tflops"]
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None

    # e2e: the public API call a user makes, target columns regenerated on
    # the device for every summand of every evaluation (as the reference's
    # _phi_block does, objective.py:561-565): a fresh oracle object per step,
    # so nothing computed by an earlier step is reused; host inputs: gate
    # matrices + directions; host output: the reduced records.
    e2e_steps = max(1, args.steps if args.e2e_steps is None else args.e2e_steps)

    def e2e_step():
        gates_host = np.ascontiguousarray(circ.gate_stack())
        dirs_host = np.ascontiguousarray(np.stack(X))
        target = make_target(spec, T_EVOL)
        r, h = gf.gradient_and_hvp(circ.with_gates(list(gates_host)), target, list(dirs_host), **kw)
        return r, h, gates_host, dirs_host

    e2e_step()  # untimed warm-up (first launches of the oracle kernels)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(e2e_steps):
        rep_e, hv_e, gates_host, dirs_host = e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks(e0.elapsed_time(e1), dist)
    e2e_val = summands * e2e_steps / (e2e_ms * 1e-3)
    rec_bytes = (2 + 64 * circ.num_logical) * 8 * nchunks
    h2d = gates_host.nbytes + dirs_host.nbytes
    # consistency: same objective from both paths
    assert abs(rep_e.value - rep.value) <= 1e-10 * max(1.0, abs(rep.value)), (rep_e.value, rep.value)

    # the same evaluation with the light-cone rule off (every slot applied to
    # every tile, as the reference applies it to the whole vector): the results
    # must agree -- the rule only skips exact zeros -- and its rate is reported
    no_lc = None
    if rank == 0 and world == 1 and os.environ.get("GF_LIGHTCONE", "1") != "0" and not args.no_lightcone_check:
        os.environ["GF_LIGHTCONE"] = "0"
        try:
            rep0, hv0 = gf.gradient_and_hvp(circ, cache, X, **kw)  # plan + warm-up
            torch.cuda.synchronize()
            e0.record(stream)
            rep0, hv0 = gf.gradient_and_hvp(circ, cache, X, **kw)
            e1.record(stream)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("GF_LIGHTCONE", None)
        ms0 = e0.elapsed_time(e1)
        g1, g0 = np.stack(rep.holomorphic_derivatives), np.stack(rep0.holomorphic_derivatives)
        h1, h0 = np.stack(hv), np.stack(hv0)
        dev_g = float(np.abs(g1 - g0).max() / np.abs(g0).max())
        dev_h = float(np.abs(h1 - h0).max() / np.abs(h0).max())
        dev_v = abs(rep.value - rep0.value) / max(1.0, abs(rep0.value))
        assert max(dev_g, dev_h, dev_v) < 1e-10, (dev_v, dev_g, dev_h)
        no_lc = {"value": summands / (ms0 * 1e-3), "unit": UNIT, "ms_per_step": ms0,
                 "max_rel_dev_vs_light_cone": {"value": dev_v, "gradient": dev_g, "hvp": dev_h},
                 "note": "GF_LIGHTCONE=0: every slot applied to every tile; one timed step"}

    del cache
    obj._PLANS.clear()
    torch.cuda.empty_cache()
    gate_sweep = None
    cpu = None
    c5 = None
    if rank == 0 and world == 1:
        if not args.no_sweep:
            gate_sweep = gate_apply_sweep(gf, peak)
        if not args.no_c5:
            c5 = c5_summand(gf, peaks64)
        if not args.no_cpu:
            from oracle import gf_oracle as O

            cores = os.cpu_count() or 1
            srng = np.random.default_rng(11)
            js = np.sort(srng.choice(TOTAL, size=REF_SAMPLE, replace=False)).astype(np.int64)
            phi = torch.empty((REF_SAMPLE, N), dtype=torch.complex128, device="cuda")
            oracle.phi0_into(torch.from_numpy(js).cuda(), None, phi)
            ph = phi.cpu().numpy()
            del phi
            t1, t2, lid = circ.slot_arrays()
            oplan = O.Plan(K_QUBITS, np.stack([t1, t2], 1), lid, circ.gate_stack())
            dt, _ = port_grad_hvp(oplan, X, js, ph, cores)
            cpu = {"value": REF_SAMPLE / dt, "unit": UNIT, "cores": cores, "kind": "port",
                   "sample": f"{REF_SAMPLE} seeded c2 summands, gradient + HVP each (oracle/gf_oracle.c, restating "
                             f"reference objective.py:322-337, 432-482) on {cores} threads, phi0 precomputed",
                   "gate_apply": cpu_gate_apply()}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "c128",
            "data": "synthetic: BASELINE configs[1] circuit (spinful FH L=8 open, 5 layers, Haar seed 1); target "
                    "columns conj(exp(-iHt)|j>) (J=1, U=4, t=0.25) computed on device by the %s oracle" % args.oracle,
            "config": CONFIG,
            "step": f"one full-sum evaluation: {summands} summands (value + gradient + HVP each), batch {batch}, "
                    f"chunk {chunk}, sharded over {world} rank(s) ({args.backend})",
            "full_sum_evals_per_s": value / TOTAL,
            "engine": dict(plan_shape, batch=batch, chunk=chunk, oracle_setup_s=round(oracle_setup_s, 3),
                           l2="inputs larger than L2 (phi0 cache %d MiB per GPU; workspace 3 x batch x 1 MiB)" %
                              ((p1 - p0) * N * 16 >> 20)),
            "roofline": {"bound": "tensor",
                         "kernel": (rev1["kernel"] if (rev1 and dom == "reverse") else
                                    f"k_fused ({dom} sweep: fused tile passes, FP64 DMMA)"),
                         "dominant_launch": rev1,
                         "sweep_executed_tflops": phases[dom]["fp64_tflops"],
                         "achieved": achieved, "peak": peaks64["dmma_tflops"], "unit": "TFLOP/s",
                         "frac": round(achieved / peaks64["dmma_tflops"], 4), "traffic": traffic,
                         "peak_source": "measured in this run: back-to-back DMMA.8x8x4 on all SMs "
                                        "(MEASURED_PEAKS.json and the profiling recipe give no FP64 peak)",
                         "fp64_fma_peak_tflops": peaks64["dfma_tflops"],
                         "algorithmic_tflops": phases[dom]["fp64_tflops_algorithmic"],
                         "live_fraction": phases[dom]["live_fraction"],
                         "algorithmic_flops": "32 flop per amplitude per dense gate / hole (SURVEY 8(d) units); "
                                              "reverse sweep 6, ascending 5, forward 1 per slot; x 2^16 amplitudes x "
                                              "36 slots x summands.  `achieved` is the dominant launch (the "
                                              "reverse sweep's first pass: every tile live, executed = algorithmic "
                                              "flops over its CUDA-event time); sweep_executed_tflops counts the "
                                              "flops the whole sweep executes (it skips the tiles outside the basis "
                                              "state's light cone, psi = 0 there: live_fraction of the slot work); "
                                              "algorithmic_tflops counts the full-vector passes of the reference",
                         "hbm_view": {"peak_gbs": peak, "peak_source": peak_src,
                                      "note": "HBM bytes per fused pass = 32 B x vectors touched x amplitudes; the "
                                              "fused sweeps make ~5 HBM round trips per 36 slots, so they are not "
                                              "HBM-bound; the standalone gate apply is (gate_apply)"}},
            "phases": phases,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(rec_bytes),
                    "full_sum_evals_per_s": e2e_val / TOTAL,
                    "path": "gf.gradient_and_hvp(circuit, %s(spec, t), directions), oracle constructed per step: every "
                            "target column regenerated on device each evaluation" % type(oracle).__name__},
            "gpu_launches": launches_all,
            "clocks": clocks,
            "no_light_cone": no_lc,
            "gate_apply": gate_sweep,
            "c5": c5,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: CPU test of the multi-rank path on one GPU)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--oracle", default="blocks", choices=["blocks", "chebyshev"],
                    help="target oracle: number-block Chebyshev (default) or full-space Chebyshev")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-lightcone-check", action="store_true")
    ap.add_argument("--summands", type=int, default=None,
                    help="profiling only: restrict each step to the first S basis states")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
