#!/usr/bin/env python
"""The reference's ``gatefit bench`` harness (reference cli.py:410-522) on the
B200 engine: the same kinds (kernels / gradient / hessian / scaling), the same
arguments and the same ``bench-v1`` CSV schema (cli.py:36, cli.py:514-521),
so its rows line up with the reference's machine-local benchmark files.

GPU-side differences, all additive:

* kernel rows are timed with CUDA events on device-resident vectors (median
  of ``--repeats``); every ``*_seconds`` row has a ``*_gbs`` companion
  (algorithmic bytes: 32 B per amplitude for a gate, 32 B per amplitude for a
  hole contraction, 16 (1 + A) B per amplitude for a hole apply, 32 A B per
  amplitude for an array gate, 16 (1 + A) B per amplitude for an array
  contraction);
* the kernel kind adds the array kernels the reference leaves unbenched
  (apply_gate_to_array, hole_contract_array) and the one-qubit gate;
* ``hessian`` takes ``--method pairs|columns`` (objective.full_hessian);
* ``scaling`` runs the basis sum on 1..N GPUs (torchrun ranks; ``--workers``
  are GPU counts) and checks bit-identical results, like the reference's
  worker-count determinism check (cli.py:485-510).

  python bench_v1.py kernels --qubits 20,24,28 --out profiles/r02
  python bench_v1.py gradient --qubits 12,16 --layers 5
  python bench_v1.py hessian --qubits 12 --bench-dedup --method pairs
"""

from __future__ import annotations

import argparse
import csv
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BENCH_SCHEMA = "bench-v1"  # reference cli.py:36
FIELDS = ["schema", "kind", "qubits", "layers", "slots", "workers", "dedup", "metric", "value"]


class IdentityOracle:
    """U = I (reference cli.py's _IdentityOracle): phi0_j = |j>, built on the
    device."""

    def __init__(self, k):
        self.num_qubits = k

    def apply(self, state):
        return np.asarray(state, np.complex128).copy()

    apply_adjoint = apply

    def phi0_into(self, js_full, sector, out):
        import torch

        out.zero_()
        idx = js_full if sector is None else (js_full >> 1)
        out[torch.arange(out.shape[0], device=out.device), idx] = 1.0


def _events_median(fn, repeats):
    import torch

    stream = torch.cuda.current_stream()
    fn()  # warm
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.median(times)


def _wall_median(fn, repeats):
    import torch

    times = []
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    return statistics.median(times)


def kernel_rows(ks, repeats, seed):
    """reference _bench_rows_kernels (cli.py:424-441) on device tensors."""
    import torch

    import paper_2506_23775_b200 as gf

    L = gf._lib
    st = L.stream_ptr()
    rng = np.random.default_rng(seed)
    rows = []
    for k in ks:
        N = 1 << k
        g = np.ascontiguousarray(gf.manifold.random_unitary(4, rng))
        g1 = np.ascontiguousarray(gf.manifold.random_unitary(2, rng))
        psi = torch.randn(N, dtype=torch.complex128, device="cuda")
        out = torch.empty_like(psi)
        hole = torch.empty(16, dtype=torch.complex128, device="cuda")
        sup = np.arange(16, dtype=np.int64)
        cases = {
            "apply_gate_adjacent": (lambda: L.check(L.lib.gf_apply_gate(psi.data_ptr(), out.data_ptr(), k, 0, 1,
                                                                        g.ctypes.data, 0, 1, st)), 32.0 * N),
            "apply_gate_general": (lambda: L.check(L.lib.gf_apply_gate(psi.data_ptr(), out.data_ptr(), k, 0, k - 1,
                                                                       g.ctypes.data, 0, 1, st)), 32.0 * N),
            "apply_gate_1q": (lambda: L.check(L.lib.gf_apply_gate_1q(psi.data_ptr(), out.data_ptr(), k, 0,
                                                                     g1.ctypes.data, 1, st)), 32.0 * N),
            "hole_contract": (lambda: L.check(L.lib.gf_hole_contract(psi.data_ptr(), psi.data_ptr(), k, 0, 1, 1,
                                                                     hole.data_ptr(), st)), 32.0 * N),
        }
        A = 16
        if 16 * N * A <= 16 << 30:  # hole arrays [2^k, 16] up to 16 GiB
            arr = torch.empty((N, A), dtype=torch.complex128, device="cuda")
            arr2 = torch.empty_like(arr)
            outT = torch.empty((A, 16), dtype=torch.complex128, device="cuda")
            cases["hole_apply"] = (lambda: L.check(L.lib.gf_hole_apply(psi.data_ptr(), arr.data_ptr(), k, 0, 1,
                                                                       sup.ctypes.data, A, st)), 16.0 * N * (1 + A))
            cases["apply_gate_to_array"] = (lambda: L.check(L.lib.gf_apply_gate_to_array(
                arr.data_ptr(), arr2.data_ptr(), k, A, 0, 1, g.ctypes.data, 0, st)), 32.0 * N * A)
            cases["hole_contract_array"] = (lambda: L.check(L.lib.gf_hole_contract_array(
                psi.data_ptr(), arr.data_ptr(), k, A, 0, 1, sup.ctypes.data, 16, outT.data_ptr(), st)),
                16.0 * N * (1 + A))
        for name, (fn, nbytes) in cases.items():
            s = _events_median(fn, repeats)
            rows.append((k, f"{name}_seconds", s))
            rows.append((k, f"{name}_gbs", nbytes / s / 1e9))
        del psi, out
        torch.cuda.empty_cache()
    return rows


def _random_bench_circuit(gf, k, layers, rng):
    """reference cli.py:444-446: periodic brick wall, one Haar gate per layer."""
    gates = [gf.manifold.random_unitary(4, rng) for _ in range(layers)]
    return gf.build_brickwall(k, layers, gates, periodic=True)


def main(argv=None):
    ap = argparse.ArgumentParser(prog="bench_v1", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("kind", choices=["kernels", "gradient", "hessian", "scaling"])
    ap.add_argument("--qubits", type=lambda s: [int(x) for x in s.split(",")], default=[4, 6, 8])
    ap.add_argument("--layers", type=int, default=5)
    ap.add_argument("--workers", type=lambda s: [int(x) for x in s.split(",")], default=[1])
    ap.add_argument("--bench-workers", type=int, default=1)
    ap.add_argument("--bench-dedup", action="store_true")
    ap.add_argument("--method", choices=["pairs", "columns"], default=None)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--inits", type=int, default=5)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)

    import torch

    import paper_2506_23775_b200 as gf

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    rows = []
    rng = np.random.default_rng(args.seed)
    if args.kind == "kernels":
        for k, metric, value in kernel_rows(args.qubits, args.repeats, args.seed):
            rows.append({"kind": "kernels", "qubits": k, "layers": "", "slots": "", "workers": 1, "dedup": "",
                         "metric": metric, "value": repr(float(value))})
    elif args.kind in ("gradient", "hessian"):
        for k in args.qubits:
            oracle = IdentityOracle(k)
            medians = []
            for _ in range(args.inits):
                circ = _random_bench_circuit(gf, k, args.layers, rng)
                if args.kind == "gradient":
                    fn = lambda: gf.full_gradient(circ, oracle)
                else:
                    fn = lambda: gf.full_hessian(circ, oracle, use_translation_dedup=args.bench_dedup,
                                                 method=args.method)
                fn()  # plan + warm-up
                medians.append(_wall_median(fn, args.repeats))
            med = statistics.median(medians)
            rep = fn()
            base = {"kind": args.kind, "qubits": k, "layers": args.layers, "slots": circ.num_slots,
                    "workers": args.bench_workers, "dedup": args.bench_dedup}
            rows.append(dict(base, metric="median_seconds", value=repr(med)))
            rows.append(dict(base, metric="median_seconds_per_summand", value=repr(med / 2**k)))
            for name, count in rep.pass_counts.items():
                rows.append(dict(base, metric=name, value=count))
    else:  # scaling over GPU ranks (this process is one rank under torchrun)
        import torch.distributed as dist

        k = args.qubits[0]
        circ = _random_bench_circuit(gf, k, args.layers, rng)
        oracle = IdentityOracle(k)
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        fn = lambda: gf.full_gradient(circ, oracle, distributed=world > 1)
        fn()
        med = _wall_median(fn, args.repeats)
        rep = fn()
        rows.append({"kind": "scaling", "qubits": k, "layers": args.layers, "slots": circ.num_slots,
                     "workers": world, "dedup": "", "metric": "median_seconds", "value": repr(med)})
        rows.append({"kind": "scaling", "qubits": k, "layers": args.layers, "slots": circ.num_slots,
                     "workers": world, "dedup": "", "metric": "value", "value": repr(rep.value)})
        if world > 1:
            dist.destroy_process_group()
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
    outdir = args.out or "."
    os.makedirs(outdir, exist_ok=True)
    path = os.path.join(outdir, f"bench_{args.kind}.csv")  # reference: <out>/bench.csv (one kind per file)
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=FIELDS)
        w.writeheader()
        for row in rows:
            w.writerow({"schema": BENCH_SCHEMA, **row})
    print(f"wrote {path} ({len(rows)} rows)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
