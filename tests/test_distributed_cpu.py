"""Multi-rank path on CPU: world_size-2 gloo run of the basis-sum sharding
(objective.shard_chunks), the all-gather of per-chunk records
(objective.gather_records) and the ordered chunk sum (objective.ordered_sum).
Chunk records are produced here by the CPU oracle (the GPU engine produces the
same record layout, include/gatefit_b200.h gf_plan_eval); the test checks that
the sharded result is bit-identical to the single-process one and equal to the
reference golden values -- the reference's worker-count determinism
(pkg/tests/test_objective.py:352-366) carried over to GPU counts."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import ROOT, golden  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _records(chunk_lo, chunk_hi, chunk):
    """Chunk records (value, D, H per logical) of BASELINE configs[0] via the oracle."""
    import sys

    sys.path.insert(0, ROOT)
    from oracle import gf_oracle as O

    g = golden("c1")
    terms, _ = O.spinful_terms(4, 1.0, 4.0, False)
    U = O.dense_target(8, terms, 0.25)
    plan = O.Plan(8, g["targets"], g["logical"], g["gates"])
    phi = O.dense_phi0(U)
    recs = []
    for c in range(chunk_lo, chunk_hi):
        js = np.arange(c * chunk, (c + 1) * chunk)
        v, d, _ = O.gradient_sum(plan, js, phi)
        h, _ = O.hvp_sum(plan, list(g["direction"]), js, phi)
        rec = np.concatenate([[v.real, v.imag], plan.logical_sum(d).reshape(-1).view(np.float64),
                              plan.logical_sum(h).reshape(-1).view(np.float64)])
        recs.append(rec)
    return torch.from_numpy(np.array(recs))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2506_23775_b200 import objective as obj

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    chunk, nchunks = 16, 16
    lo, hi = obj.shard_chunks(nchunks, rank, world)
    local = _records(lo, hi, chunk)
    allrec = obj.gather_records(local, lo, nchunks, rank, world, dist)
    tot = obj.ordered_sum(allrec.numpy())
    np.save(os.path.join(out, f"rank{rank}.npy"), tot)
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_bit_identical(tmp_path):
    import torch.multiprocessing as mp

    from paper_2506_23775_b200 import objective as obj

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    single = obj.ordered_sum(_records(0, 16, 16).numpy())
    assert np.array_equal(r0, r1) and np.array_equal(r0, single)
    g = golden("c1")
    assert abs(-r0[0] - g["value"]) < 1e-12
    d = r0[2:2 + 96].view(np.complex128).reshape(3, 4, 4)
    h = r0[2 + 96:].view(np.complex128).reshape(3, 4, 4)
    assert np.abs(d - g["holo"]).max() < 1e-12 * np.abs(g["holo"]).max()
    assert np.abs(h - g["hvp"]).max() < 1e-12 * np.abs(g["hvp"]).max()
