"""Randomised check of the light-cone rule (dead tiles skipped in all three
sweeps): random circuits -- random slot pairs incl. long-range and swapped
targets, shared logical gates, random depth -- at forced small tiles (many
global bits, many passes), full space and parity sectors, one and three HVP
directions.  Compares GF_LIGHTCONE=1 with GF_LIGHTCONE=0 and with the streaming
engine (one launch per slot on the whole vector).
  python tools/stress_lightcone.py [cases]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_23775_b200 as gf  # noqa: E402
from paper_2506_23775_b200 import manifold, objective as obj  # noqa: E402
from paper_2506_23775_b200.circuit import Circuit, GateSlot  # noqa: E402
from paper_2506_23775_b200.kernels import Gate  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))


def run(circ, orc, X, env, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        rep, hv = gf.gradient_and_hvp(circ, orc, X[0], parity_mode=kw.pop("parity"), **kw)
        multi = gf.hessian_vector_products(circ, orc, X, **{k: v for k, v in kw.items() if k != "fold"})
        live = list(obj._PLANS.values())[-1].describe()["live_fraction"]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return rep.value, np.stack(rep.holomorphic_derivatives), np.stack(hv), np.stack([np.stack(m) for m in multi]), live


def main(cases):
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2024)
    worst = 0.0
    for case in range(cases):
        k = int(rng.integers(8, 14))
        parity = bool(rng.integers(0, 2))
        nlog = int(rng.integers(1, 5))
        nslots = int(rng.integers(3, 3 * k))
        gates = []
        for _ in range(nlog):
            if parity:
                m = manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng))
            else:
                m = manifold.random_unitary(4, rng)
            gates.append(Gate(m, (0, 1), parity_sparse=parity))
        slots = []
        for _ in range(nslots):
            a, b = rng.choice(k, size=2, replace=False)
            if rng.random() < 0.6:  # mostly short-range, some swapped
                b = (a + 1) % k if rng.random() < 0.8 else (a - 1) % k
            slots.append(GateSlot(int(rng.integers(0, nlog)), (int(a), int(b))))
        circ = Circuit(k, slots, gates)
        u = manifold.random_unitary(1 << k, rng) if k <= 10 else None
        if u is None:
            spec = gf.build_spinful_fh(k // 2, 1.0, 4.0, True) if k % 2 == 0 else None
            if spec is None:
                continue
            orc = gf.ChebyshevOracle(spec, 0.25)
        else:
            if parity:  # a parity-conserving target keeps sector sums meaningful; any target works for the check
                pass
            orc = gf.DenseOracle.from_matrix(u)
        X = [[manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
              for g in gates] for _ in range(3)]
        sector = (None if not parity else int(rng.integers(0, 2)))
        K = k - (1 if sector is not None else 0)
        m = str(int(rng.integers(6, min(11, K) + 1)))
        nsum = min(1 << K, 48)
        basis = np.sort(rng.choice(1 << K, size=nsum, replace=False)).astype(np.int64)
        kw = dict(parity=parity, sector=sector, basis=(basis, None))
        on = run(circ, orc, X, {"GF_LIGHTCONE": "1", "GF_FUSED_M": m}, **dict(kw))
        off = run(circ, orc, X, {"GF_LIGHTCONE": "0", "GF_FUSED_M": m}, **dict(kw))
        st = run(circ, orc, X, {"GF_ENGINE": "stream"}, **dict(kw))
        errs = [abs(on[0] - off[0]) / max(1.0, abs(off[0])), rel(on[1], off[1]), rel(on[2], off[2]), rel(on[3], off[3]),
                abs(on[0] - st[0]) / max(1.0, abs(st[0])), rel(on[1], st[1]), rel(on[2], st[2]), rel(on[3], st[3])]
        worst = max(worst, max(errs))
        flag = "" if max(errs) < 1e-10 else "   <-- MISMATCH"
        print(f"case {case:3d} k={k:2d} parity={int(parity)} sector={sector} m={m:>2s} slots={nslots:3d} nlog={nlog} "
              f"live={on[4]['forward']:.3f}/{on[4]['reverse']:.3f} max err {max(errs):.2e}{flag}", flush=True)
        obj._PLANS.clear()
    print("worst", worst)
    return 0 if worst < 1e-10 else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 40))
