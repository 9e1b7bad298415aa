"""CPU tests of the host-side mirror of the reference API (no GPU needed):
manifold math, circuit bookkeeping, models, tCG, Hessian blocks, chunking --
each checked against fixtures from the unmodified reference or against the
reference's own property tests (pkg/tests/test_manifold.py, test_circuit.py,
test_models.py, test_optimizer.py)."""

import math

import numpy as np
import pytest

from conftest import ROOT, golden, rel_err
from paper_2506_23775_b200 import circuit as C
from paper_2506_23775_b200 import manifold as M
from paper_2506_23775_b200 import models, objective, optimizer
from paper_2506_23775_b200.kernels import Gate


def test_riemannian_conversion_matches_reference_c1():
    g = golden("c1")
    for v, d, e, r in zip(g["gates"], g["holo"], g["euclid"], g["riem"]):
        eu = M.euclid_gradient_from_holomorphic(d)
        assert np.array_equal(eu, e)
        assert rel_err(M.project_tangent_gate(v, eu), r) < 1e-14


def test_hessian_apply_matches_reference_c1():
    g = golden("c1")
    hx = [M.hessian_apply_gate(v, e, M.euclid_gradient_from_holomorphic(h), x)
          for v, e, h, x in zip(g["gates"], g["euclid"], g["hvp"], g["direction"])]
    assert rel_err(np.stack(hx), g["hess_x"]) < 1e-13
    assert abs(sum(M.inner(x, y) for x, y in zip(g["direction"], hx)) - g["x_hess_x"]) < 1e-12


def test_hessian_blocks_apply_direction_equals_reference_hvp():
    g = golden("c1")
    keys = [tuple(int(v) for v in k) for k in g["hess_keys"]]
    hb = objective.HessianBlocks(3, g["hess_support"], dict(zip(keys, g["hess_blocks"])))
    out = hb.apply_direction(list(g["direction"]))
    assert rel_err(np.stack(out), g["hvp"]) < 1e-12


def test_random_unitary_reproduces_reference_draws():
    g = golden("c1")
    spec, circ, rng = models.spinful_layer_circuit(4, 3, False, seed=0)
    assert np.array_equal(circ.gate_stack(), g["gates"])
    assert [s.targets for s in circ.slots] == [tuple(t) for t in g["targets"]]


def test_manifold_properties(rng):
    v = M.random_unitary(4, rng)
    x = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    t = M.project_tangent(v, x)
    assert np.allclose(M.project_tangent(v, t), t, atol=1e-14)
    r = M.retract_polar(v, 0.1 * t)
    assert np.allclose(r.conj().T @ r, np.eye(4), atol=1e-13)
    assert np.allclose(M.retract_polar(v, np.zeros((4, 4))), v, atol=1e-14)
    with pytest.raises(M.DegenerateRetractionError):
        M.retract_polar(np.eye(4), -np.eye(4))
    p = M.parity_join(M.random_unitary(2, rng), M.random_unitary(2, rng))
    o, e = M.parity_split(p)
    assert np.array_equal(M.parity_join(o, e), p)
    with pytest.raises(ValueError):
        M.parity_split(v)
    rp = M.retract_gate(p, M.project_tangent_gate(p, x, True), parity=True)
    assert np.all(rp.reshape(16)[[1, 2, 4, 7, 8, 11, 13, 14]] == 0)


def test_translation_classes_match_reference():
    g = golden("dedup")
    rng = np.random.default_rng(7)
    gates = [M.random_unitary(4, rng) for _ in range(3)]
    circ = C.build_brickwall(6, 3, gates, periodic=True)
    assert np.array_equal(circ.gate_stack(), g["gates"])
    got = np.array([[a, b, m] for (a, b), m in C.translation_classes(circ)])
    assert np.array_equal(got, g["classes"])
    alt = C.translation_classes(circ, policy="lex_max")
    assert sorted(m for _, m in alt) == sorted(int(x) for x in g["classes"][:, 2])
    with pytest.raises(ValueError):
        C.translation_classes(C.build_brickwall(6, 2, gates[:2], periodic=False))


def test_accumulate_shared_and_validation(rng):
    circ = C.build_brickwall(4, 2, [M.random_unitary(4, rng) for _ in range(2)], periodic=True)
    grads = [rng.normal(size=(4, 4)) for _ in range(circ.num_slots)]
    acc = C.accumulate_shared(grads, circ)
    want = [sum(gr for s, gr in zip(circ.slots, grads) if s.logical_id == l) for l in range(2)]
    assert all(np.allclose(a, w) for a, w in zip(acc, want))
    with pytest.raises(ValueError):
        C.Circuit(3, [C.GateSlot(0, (0, 0))], [Gate(np.eye(4), (0, 1))])
    with pytest.raises(ValueError):
        C.build_brickwall(3, 1, [np.eye(4)])


def test_models_match_reference():
    g = golden("models")
    for L, periodic in ((4, False), (4, True), (8, False), (12, False), (14, True), (16, True)):
        key = f"spinful_L{L}_{'p' if periodic else 'o'}"
        spec = models.build_spinful_fh(L, 1.0, 4.0, periodic)
        arr = np.array([[t.sites[0], t.sites[1], t.coefficient, t.operator == "hop"] for t in spec.terms], float)
        assert np.array_equal(arr, g[key + "_terms"])
        assert [len(x.bonds) for x in spec.trotter_groups] == list(g[key + "_groups"])
    assert rel_err(models.dense_hamiltonian(models.build_spinful_fh(2, 1.0, 4.0, False)), g["spinful_L2_H"]) == 0
    spec = models.build_spinless_fh(6, 1.0, 4.0, True)
    circ = models.build_trotter_circuit(spec, models.TrotterPlan(4, 1, 0.3))
    assert circ.num_logical == int(g["trotter4_spinless6_ngates"])
    assert rel_err(circ.gate_stack(), g["trotter4_spinless6_gates"]) < 1e-14
    assert [s.targets for s in circ.slots] == [tuple(t) for t in g["trotter4_spinless6_targets"]]


def test_dense_oracle_host_apply_matches_reference():
    g = golden("models")
    o = models.DenseOracle(models.build_spinful_fh(3, 1.0, 4.0, True), 0.25)
    assert rel_err(o.apply(g["krylov_in"]), g["dense_out"]) < 1e-12


def test_truncated_cg_behaviour(rng):
    grad = [rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)) for _ in range(2)]
    # identity Hessian, large radius: the Newton step -g
    step, reason, it = optimizer.truncated_cg(lambda xs: [x.copy() for x in xs], grad, 1e3, optimizer.TcgParams())
    assert reason == "converged" and all(np.allclose(s, -g) for s, g in zip(step, grad))
    # negative curvature ends on the boundary
    step, reason, _ = optimizer.truncated_cg(lambda xs: [-x for x in xs], grad, 0.5, optimizer.TcgParams())
    assert reason == "negative_curvature"
    assert abs(math.sqrt(sum(np.vdot(s, s).real for s in step)) - 0.5) < 1e-12
    z, reason, it = optimizer.truncated_cg(lambda xs: xs, [np.zeros((4, 4))], 1.0, optimizer.TcgParams())
    assert reason == "zero_gradient" and it == 0
    with pytest.raises(FloatingPointError):
        optimizer.truncated_cg(lambda xs: [x * np.nan for x in xs], grad, 1.0, optimizer.TcgParams())
    with pytest.raises(ValueError):
        optimizer.TrustRegionParams(accept_threshold=0.5, shrink_threshold=0.25)


def test_chunk_bounds_partition(rng):
    for _ in range(20):
        total = int(rng.integers(1, 5000))
        nch = int(rng.integers(1, 80))
        cover = [i for a, b in objective.chunk_bounds(total, nch) for i in range(a, b)]
        assert cover == list(range(total))
    assert objective.chunk_bounds(0) == []
    assert objective.parallel_reduce(1000, lambda a, b: sum(range(a, b)), 4) == sum(range(1000))


def test_shard_chunks_cover_exactly():
    for nchunks in (1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [objective.shard_chunks(nchunks, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nchunks
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_bench_reference_arm_uses_the_same_c2_workload():
    """bench.py --impl reference reads the circuit and direction from the
    reference-written c2_slice fixture (it must not import the product); they
    must equal the B200 arm's recipe bit for bit (same config in both arms)."""
    import bench

    gf, spec, circ, X = bench.workload()
    g = golden("c2_slice")
    t1, t2, lid = circ.slot_arrays()
    assert np.array_equal(np.stack([t1, t2], 1), g["targets"])
    assert np.array_equal(lid, g["logical"])
    assert np.array_equal(circ.gate_stack(), g["gates"])
    assert np.array_equal(np.stack(X), g["direction"])
    assert int(g["k"]) == bench.K_QUBITS


def test_bench_reference_arm_does_not_import_the_product(tmp_path):
    """The reference arm runs the oracle port only: no paper_2506_23775_b200
    module (and so no libgfcuda.so) may be loaded by it."""
    import subprocess
    import sys

    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0'];"
            "import bench; bench.REF_SAMPLE=4; bench.run_reference(bench.argparse.Namespace(gpus=1, steps=1, "
            "warmup=0)); assert not any(m.startswith('paper_2506_23775_b200') for m in sys.modules), "
            "[m for m in sys.modules if m.startswith('paper')]; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok")
