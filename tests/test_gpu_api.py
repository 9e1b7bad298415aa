"""The reference's own behavioural tests (pkg/tests/test_kernels.py,
test_objective.py, test_optimizer.py, test_models.py) restated against the
GPU drop-in API.  Run with ``pytest -m gpu``."""

import itertools

import numpy as np
import pytest

from conftest import golden, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2506_23775_b200 as gf  # noqa: E402
from paper_2506_23775_b200 import kernels as K  # noqa: E402
from paper_2506_23775_b200 import manifold  # noqa: E402
from oracle import gf_oracle as O  # noqa: E402


def dense_two_qubit(mat, t1, t2, k):
    """Independent dense embedding by basis-pair enumeration (reference
    tests/conftest.py:16-36 restated)."""
    N = 2**k
    out = np.zeros((N, N), dtype=complex)
    others = [q for q in range(k) if q not in (t1, t2)]
    for x in range(N):
        for y in range(N):
            if any(((x >> (k - 1 - q)) & 1) != ((y >> (k - 1 - q)) & 1) for q in others):
                continue
            xi = 2 * ((x >> (k - 1 - t1)) & 1) + ((x >> (k - 1 - t2)) & 1)
            yi = 2 * ((y >> (k - 1 - t1)) & 1) + ((y >> (k - 1 - t2)) & 1)
            out[x, y] = mat[xi, yi]
    return out


def dense_circuit(circ):
    U = np.eye(2**circ.num_qubits, dtype=complex)
    for s in circ.slots:
        U = dense_two_qubit(circ.logical_gates[s.logical_id].matrix, *s.targets, circ.num_qubits) @ U
    return U


def random_circuit(k, n, rng):
    gates, slots = [], []
    for i in range(n):
        t1, t2 = (int(x) for x in rng.choice(k, size=2, replace=False))
        gates.append(gf.Gate(manifold.random_unitary(4, rng), (t1, t2)))
        slots.append(gf.GateSlot(i, (t1, t2)))
    return gf.Circuit(k, slots, gates)


def random_tangent(v, rng):
    return manifold.project_tangent(v, rng.normal(size=v.shape) + 1j * rng.normal(size=v.shape))


def brickwall(k, layers, rng, periodic=True):
    return gf.build_brickwall(k, layers, [manifold.random_unitary(4, rng) for _ in range(layers)], periodic=periodic)


class MatrixOracle:
    def __init__(self, u):
        self.num_qubits = int(np.log2(u.shape[0]) + 0.5)
        self.matrix = u

    def apply(self, s):
        return self.matrix @ s

    def apply_adjoint(self, s):
        return self.matrix.conj().T @ s


# ------------------------------------------------------------------ kernels


COUNTS = ("gate_applications", "array_gate_applications", "hole_applications", "hole_contractions",
          "pair_contractions")


def test_dense_oracle_equivalence_exhaustive_basis():
    """test_kernels.py:49-63: every ordered target pair, every basis input, k <= 4."""
    rng = np.random.default_rng(5)
    for k in (2, 3, 4):
        for t1, t2 in itertools.permutations(range(k), 2):
            g = manifold.random_unitary(4, rng)
            dense = dense_two_qubit(g, t1, t2, k)
            basis = torch.eye(2**k, dtype=torch.complex128, device="cuda")
            for j in range(2**k):
                out = K.apply_gate(basis[j].contiguous(), gf.Gate(g, (t1, t2))).cpu().numpy()
                assert np.allclose(out, dense[:, j], atol=1e-13)
                arr = K.hole_apply(np.eye(2**k)[j].astype(complex), (t1, t2))
                assert np.allclose(arr @ g.reshape(16), dense[:, j], atol=1e-13)


def test_linearity_norm_and_variants(rng):
    k = 6
    psi = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    chi = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    g = gf.Gate(manifold.random_unitary(4, rng), (1, 4))
    a, b = 0.3 - 0.7j, -1.2 + 0.1j
    assert np.allclose(K.apply_gate(a * psi + b * chi, g), a * K.apply_gate(psi, g) + b * K.apply_gate(chi, g),
                       atol=1e-13)
    n0 = np.linalg.norm(psi)
    assert abs(np.linalg.norm(K.apply_gate(psi, g)) - n0) < 1e-12 * n0
    assert np.array_equal(K.apply_gate(psi, g, variant="kernel"), K.apply_gate(psi, g, variant="plain"))
    with pytest.raises(ValueError):
        K.apply_gate(psi, g, variant="fancy")


def test_hole_contract_reinsertion_and_basis(rng):
    """test_kernels.py:106-138."""
    p = np.zeros(4, complex)
    p[0] = 1
    d = K.hole_contract(p, p, (0, 1))
    e = np.zeros((4, 4))
    e[0, 0] = 1
    assert np.allclose(d, e, atol=1e-15)
    k = 5
    bra = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    ket = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    for t in [(0, 1), (1, 3), (3, 0), (4, 2)]:
        d = K.hole_contract(bra, ket, t)
        for _ in range(3):
            g = manifold.random_unitary(4, rng)
            rhs = bra @ K.apply_gate(ket, gf.Gate(g, t))
            assert abs(np.sum(g * d) - rhs) < 1e-12 * max(1.0, abs(rhs))
    with pytest.raises(ValueError):
        K.hole_contract(bra, ket[:16], (0, 1))


def test_hole_apply_support_and_layout(rng):
    """test_kernels.py:146-173."""
    arr = K.hole_apply(np.eye(8)[0].astype(complex), (0, 1))
    assert [a for a in range(16) if np.any(arr[:, a] != 0)] == [0, 4, 8, 12]
    psi = rng.normal(size=8) + 1j * rng.normal(size=8)
    arr = K.hole_apply(psi, (1, 2))
    assert arr.flags["C_CONTIGUOUS"] and arr.shape == (8, 16)
    arrp = K.hole_apply(psi, (0, 1), support=K.PARITY_SUPPORT)
    out = K.apply_gate_to_array(arrp, gf.Gate(manifold.random_unitary(4, rng), (1, 2)))
    assert out.shape == arrp.shape


def test_array_ops_double_reinsertion_and_commuting(rng):
    """test_kernels.py:176-246."""
    k = 4
    psi = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    bra = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    g1, g2 = manifold.random_unitary(4, rng), manifold.random_unitary(4, rng)
    arr = K.hole_apply(psi, (0, 1))
    rebuilt = K.apply_gate_to_array(arr, gf.Gate(g2, (2, 3))) @ g1.reshape(16)
    direct = K.apply_gate(K.apply_gate(psi, gf.Gate(g1, (0, 1))), gf.Gate(g2, (2, 3)))
    assert np.allclose(rebuilt, direct, atol=1e-13)
    arr = K.hole_apply(psi, (1, 2))
    b = K.hole_contract_array(bra, arr, (1, 2))
    lhs = g1.reshape(16) @ b @ g1.reshape(16)
    rhs = bra @ K.apply_gate(K.apply_gate(psi, gf.Gate(g1, (1, 2))), gf.Gate(g1, (1, 2)))
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(rhs))
    assert np.all(K.hole_contract_array(np.zeros(2**k, complex), arr, (2, 3)) == 0)


# ---------------------------------------------------------------- objective


def test_j_zero_trotter_is_exact():
    """test_objective.py:41-48."""
    spec = gf.build_spinless_fh(4, 0.0, 4.0, periodic=True)
    orc = gf.make_oracle(spec, 0.7, "dense")
    for order in (1, 2):
        circ = gf.build_trotter_circuit(spec, gf.TrotterPlan(order, 1, 0.7))
        assert gf.target_value(circ, orc) == pytest.approx(-(2**4), abs=1e-10)


def test_target_value_dense_trace_and_frobenius(rng):
    """test_objective.py:51-66."""
    k = 6
    circ = random_circuit(k, 5, rng)
    u = manifold.random_unitary(2**k, rng)
    got = gf.target_value(circ, MatrixOracle(u))
    C = dense_circuit(circ)
    want = -np.real(np.trace(u.conj().T @ C))
    assert got == pytest.approx(want, abs=1e-11)
    assert gf.frobenius_error_squared(got, k) == pytest.approx(np.linalg.norm(C - u) ** 2, rel=1e-10)


def test_gradient_finite_differences(rng):
    """test_objective.py:144-156 (central differences, rel 1e-6)."""
    circ = brickwall(6, 3, rng)
    orc = gf.DenseOracle.from_matrix(manifold.random_unitary(2**6, rng))
    rep = gf.full_gradient(circ, orc)
    step = 1e-5
    for _ in range(5):
        dirs = [random_tangent(g.matrix, rng) for g in circ.logical_gates]
        plus = circ.with_gates([g.matrix + step * d for g, d in zip(circ.logical_gates, dirs)])
        minus = circ.with_gates([g.matrix - step * d for g, d in zip(circ.logical_gates, dirs)])
        fd = (gf.target_value(plus, orc) - gf.target_value(minus, orc)) / (2 * step)
        an = sum(manifold.inner(g, d) for g, d in zip(rep.per_logical_gradient, dirs))
        assert fd == pytest.approx(an, rel=1e-6)


def test_gradient_vanishes_at_representable_optimum():
    """test_objective.py:135-141."""
    spec = gf.build_spinless_fh(6, 0.0, 4.0, periodic=True)
    orc = gf.make_oracle(spec, 0.5, "dense")
    circ = gf.build_trotter_circuit(spec, gf.TrotterPlan(2, 1, 0.5))
    rep = gf.full_gradient(circ, orc)
    assert np.sqrt(sum(manifold.inner(g, g) for g in rep.per_logical_gradient)) < 1e-8


def test_phase_covariance(rng):
    """test_objective.py:159-180."""
    k, n = 6, 3
    circ = random_circuit(k, n, rng)
    u = manifold.random_unitary(2**k, rng)
    theta = 0.4
    scaled = circ.with_gates([np.exp(1j * theta) * g.matrix for g in circ.logical_gates])
    want = -np.real(np.exp(1j * n * theta) * np.trace(u.conj().T @ dense_circuit(circ)))
    assert gf.target_value(scaled, MatrixOracle(u)) == pytest.approx(want, abs=1e-11)


def test_hessian_blocks_match_entry_pair_enumeration(rng):
    """test_objective.py:183-213 on k=2 (second differences of the bilinear summand)."""
    k = 2
    circ = random_circuit(k, 2, rng)
    u = manifold.random_unitary(2**k, rng)
    rep = gf.full_hessian(circ, MatrixOracle(u))
    blk = rep.hessian.blocks[(0, 1)]
    t1, t2 = circ.slots[0].targets, circ.slots[1].targets

    def ft(m1, m2):
        return np.trace(u.conj().T @ (dense_two_qubit(m2, *t2, k) @ dense_two_qubit(m1, *t1, k)))

    g1, g2 = circ.logical_gates[0].matrix, circ.logical_gates[1].matrix
    base = ft(g1, g2)
    for a in range(16):
        for b in range(16):
            ea, eb = np.zeros(16), np.zeros(16)
            ea[a] = eb[b] = 1.0
            val = ft(g1 + ea.reshape(4, 4), g2 + eb.reshape(4, 4)) - ft(g1 + ea.reshape(4, 4), g2) \
                - ft(g1, g2 + eb.reshape(4, 4)) + base
            assert abs(blk[a, b] - val) < 1e-7


def test_hessian_dedup_and_parity_blocks_vs_reference():
    """test_objective.py:229-276: dedup equals full enumeration; parity blocks
    are the on-pattern submatrix -- against the reference fixture."""
    g = golden("dedup")
    circ = gf.Circuit(int(g["k"]), [gf.GateSlot(int(l), tuple(int(x) for x in t))
                                    for t, l in zip(g["targets"], g["logical"])],
                      [gf.Gate(m, (0, 1)) for m in g["gates"]],
                      gf.BrickwallMeta(3, tuple(int(l) for l in g["logical"]), 2, True))
    orc = gf.DenseOracle.from_matrix(g["U"])
    for tag, dedup, method in (("full_", False, "columns"), ("full_", False, "pairs"), ("dedup_", True, "pairs"),
                               ("dedup_", True, "columns")):
        rep = gf.full_hessian(circ, orc, use_translation_dedup=dedup, method=method)
        keys = [tuple(int(v) for v in kk) for kk in g[tag + "keys"]]
        assert sorted(rep.hessian.blocks) == keys
        sc = np.abs(g[tag + "blocks"]).max()
        for kk, ref in zip(keys, g[tag + "blocks"]):
            assert np.abs(rep.hessian.blocks[kk] - ref).max() < 1e-10 * sc
        assert rep.pass_counts["pair_contractions"] == int(g[tag + "counts"][4])
        if method == "pairs":
            # the reference's own algorithm: every counter equal -- with dedup
            # that is the work actually saved (fewer arrays, hole applications
            # and pair contractions than the full enumeration)
            assert [rep.pass_counts[c] for c in COUNTS] == [int(x) for x in g[tag + "counts"]]
            assert rep.engine["hessian_method"] == "pairs" and rep.engine["dedup"] == dedup
    pc = gf.Circuit(int(g["p_k"]), [gf.GateSlot(int(l), tuple(int(x) for x in t))
                                    for t, l in zip(g["p_targets"], g["p_logical"])],
                    [gf.Gate(m, (0, 1), parity_sparse=True) for m in g["p_gates"]])
    for method in ("columns", "pairs"):
        prep = gf.full_hessian(pc, gf.DenseOracle.from_matrix(g["p_U"]), parity_mode=True, method=method)
        assert len(prep.hessian.support) == 8
        assert rel_err(np.stack(prep.per_logical_gradient), g["p_riem"]) < 1e-10
        sc = np.abs(g["p_hess_blocks"]).max()
        for kk, ref in zip([tuple(int(v) for v in x) for x in g["p_hess_keys"]], g["p_hess_blocks"]):
            assert np.abs(prep.hessian.blocks[kk] - ref).max() < 1e-10 * sc


def test_hvp_zero_and_column_extraction(rng):
    """test_objective.py:279-326."""
    k = 6
    circ = random_circuit(k, 3, rng)
    orc = MatrixOracle(manifold.random_unitary(2**k, rng))
    out = gf.hessian_vector_product(circ, orc, [np.zeros((4, 4))] * 3)
    assert all(np.all(o == 0) for o in out)
    rep = gf.full_hessian(circ, orc)
    z = [np.zeros((4, 4), dtype=complex) for _ in range(3)]
    direction = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    z[1] = direction
    out = gf.hessian_vector_product(circ, orc, z)
    assert np.allclose(out[0].reshape(16), rep.hessian.blocks[(0, 1)] @ direction.reshape(16), atol=1e-10)
    assert np.allclose(out[2].reshape(16), rep.hessian.blocks[(1, 2)].T @ direction.reshape(16), atol=1e-10)
    assert np.allclose(out[1], 0, atol=1e-11)
    zz = [rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)) for _ in range(3)]
    via_blocks = rep.hessian.apply_direction(zz)
    via_pass = gf.hessian_vector_product(circ, orc, zz)
    sc = max(np.abs(np.stack(via_blocks)).max(), 1e-12)
    assert all(np.abs(a - b).max() < 1e-9 * sc for a, b in zip(via_blocks, via_pass))


def test_summand_gradient_and_pass_cache(rng):
    """test_objective.py:69-132 via the GPU gate kernels."""
    k = 5
    circ = random_circuit(k, 4, rng)
    orc = MatrixOracle(manifold.random_unitary(2**k, rng))
    value, derivs = gf.summand_gradient(2, circ, orc)
    for l, s in enumerate(circ.slots):
        g = circ.logical_gates[s.logical_id].matrix
        assert abs(np.sum(g * derivs[l]) - value) < 1e-12 * max(1.0, abs(value))
    with pytest.raises(ValueError):
        gf.summand_gradient(100, circ, orc)


def test_hamiltonian_apply_and_circuit_apply(rng):
    spec = gf.build_spinful_fh(3, 1.0, 4.0, True)
    psi = rng.normal(size=64) + 1j * rng.normal(size=64)
    assert rel_err(gf.hamiltonian_apply(spec, psi), gf.dense_hamiltonian(spec) @ psi) < 1e-13
    circ = random_circuit(6, 5, rng)
    out = gf.circuit_apply(circ, psi)
    assert rel_err(out, dense_circuit(circ) @ psi) < 1e-12
    back = gf.circuit_apply(circ, psi, "backward_transposed")
    assert rel_err(back, dense_circuit(circ).T @ psi) < 1e-12


# ---------------------------------------------------------------- optimizer


def test_optimize_monotone_unitary_and_use_hvp(rng):
    """test_optimizer.py:125-150 plus the use_hvp operator path."""
    circ = brickwall(6, 3, rng)
    orc = gf.make_oracle(gf.build_spinless_fh(6, 1.0, 4.0, periodic=True), 0.3, "dense")
    final, trace = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=6))
    accepted = [r.value for r in trace.records if r.accepted]
    f = [trace.records[0].value] + accepted
    assert all(b <= a + 1e-12 for a, b in zip(f, f[1:]))
    for g in final.logical_gates:
        assert np.allclose(g.matrix.conj().T @ g.matrix, np.eye(4), atol=1e-12)
    final2, trace2 = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=6, use_hvp=True))
    assert np.allclose([r.value for r in trace2.records], [r.value for r in trace.records], rtol=1e-8, atol=1e-9)


def test_optimize_parity_mode_keeps_sparsity_and_sector_objective():
    """test_optimizer.py:152-173, plus the same loop on the even-sector objective."""
    spec = gf.build_spinless_fh(6, 1.0, 4.0, periodic=True)
    orc = gf.make_oracle(spec, 0.3, "dense")
    circ = gf.build_trotter_circuit(spec, gf.TrotterPlan(1, 1, 0.3))
    final, trace = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=3), parity_mode=True)
    for g in final.logical_gates:
        assert np.all(g.matrix.reshape(16)[[1, 2, 4, 7, 8, 11, 13, 14]] == 0)
    final2, trace2 = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=3, use_hvp=True),
                                              parity_mode=True, sector="even")
    assert all(np.isfinite(r.value) for r in trace2.records)
    with pytest.raises(ValueError):
        rng = np.random.default_rng(0)
        gf.trust_region_optimize(brickwall(6, 2, rng), orc, parity_mode=True)


def test_optimize_dedup_matches_plain_iterates(rng):
    """test_optimizer.py:175-192."""
    circ = brickwall(6, 2, rng)
    orc = gf.make_oracle(gf.build_spinless_fh(6, 1.0, 4.0, periodic=True), 0.4, "dense")
    p = gf.TrustRegionParams(max_iterations=3)
    _, t1 = gf.trust_region_optimize(circ, orc, p)
    _, t2 = gf.trust_region_optimize(circ, orc, p, use_translation_dedup=True)
    assert np.allclose([r.value for r in t1.records], [r.value for r in t2.records], rtol=1e-10, atol=1e-10)
