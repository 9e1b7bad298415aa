"""Multi-rank basis sum on the GPU: ``distributed=True`` evaluations in two
processes that share cuda:0 over gloo (this pool has one GPU per box; the
ranks never wait on each other's kernels, only on the end-of-evaluation
all-gather of per-chunk records).  The result must be bit-identical to the
single-process evaluation -- the reference's worker-count determinism
(objective.py:513-533, pkg/tests/test_objective.py:352-366) carried over to
GPU counts -- and ``bench.py --gpus 2 --backend gloo`` must run end to end."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA GPU", allow_module_level=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name):
    import paper_2506_23775_b200 as gf

    if name == "c1":
        g = golden("c1")
        spec, circ, _ = gf.spinful_layer_circuit(4, 3, False, seed=0)
        circ = circ.with_gates(list(g["gates"]))
        return circ, gf.DenseOracle(spec, 0.25), list(g["direction"]), {}
    # c2 slice: 1024 seeded summands (16 chunks of 64), two batches of 512
    g = golden("c2_slice")
    spec, circ, _ = gf.spinful_layer_circuit(8, 5, False, seed=1)
    idx = np.sort(np.random.default_rng(9).choice(1 << 16, size=1024, replace=False)).astype(np.int64)
    return circ, gf.NumberBlockOracle(spec, 0.25), list(g["direction"]), {"basis": (idx, None), "batch": 512}


def _evaluate(name, distributed):
    import paper_2506_23775_b200 as gf

    circ, orc, X, kw = _case(name)
    rep, hv = gf.gradient_and_hvp(circ, orc, X, distributed=distributed, **kw)
    return np.concatenate([[rep.value], np.stack(rep.holomorphic_derivatives).reshape(-1).view(np.float64),
                           np.stack(hv).reshape(-1).view(np.float64)])


def _worker(rank, world, port, name, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = _evaluate(name, True)
    np.save(os.path.join(out, f"{name}_rank{rank}.npy"), res)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c2slice"])
def test_two_rank_evaluation_bit_identical_to_one(tmp_path, name):
    import torch.multiprocessing as mp

    single = _evaluate(name, False)
    mp.spawn(_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / f"{name}_rank0.npy")
    r1 = np.load(tmp_path / f"{name}_rank1.npy")
    assert np.array_equal(r0, r1)
    assert np.array_equal(r0, single)
    if name == "c1":
        g = golden("c1")
        assert abs(r0[0] - g["value"]) < 1e-12


def test_bench_two_ranks_gloo_end_to_end():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--summands", "1024",
           "--batch", "256", "--steps", "1", "--warmup", "1", "--e2e-steps", "1", "--no-sweep", "--no-cpu",
           "--no-c5"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
