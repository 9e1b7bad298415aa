"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
and the reference's golden fixtures.  Run with ``pytest -m gpu``."""

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

TOL = 1e-10  # north-star tolerance for cost / gradient / HVP (fp64)


def _loaded_libs():
    with open("/proc/self/maps") as fh:
        return fh.read()


def test_native_library_is_loaded():
    assert "libgfcuda.so" in _loaded_libs()


# ----------------------------------------------------------------- kernels


def test_kernels_match_reference_vectors():
    g = golden("kernels")
    psi, bra = g["psi"], g["bra"]
    for i, t in enumerate(g["pairs"]):
        t = tuple(int(x) for x in t)
        t2 = tuple(int(x) for x in g["second_pairs"][i])
        assert rel_err(K.apply_gate(psi, K.Gate(g["gates"][i], t)), g["apply"][i]) < 1e-14
        assert rel_err(K.apply_gate(psi, K.Gate(g["pgates"][i], t)), g["apply_parity"][i]) < 1e-14
        assert rel_err(K.hole_contract(bra, psi, t), g["hole_contract"][i]) < 1e-13
        arr = K.hole_apply(psi, t)
        assert np.array_equal(arr, g["hole_apply"][i])
        assert np.array_equal(K.hole_apply(psi, t, K.PARITY_SUPPORT), g["hole_apply_parity"][i])
        assert rel_err(K.apply_gate_to_array(arr, K.Gate(g["gates"][i], t2)), g["array_apply"][i]) < 1e-14
        assert rel_err(K.hole_contract_array(bra, arr, t2), g["hole_contract_array"][i]) < 1e-13
        arrp = K.hole_apply(psi, t, K.PARITY_SUPPORT)
        assert rel_err(K.hole_contract_array(bra, arrp, t2, K.PARITY_SUPPORT),
                       g["hole_contract_array_parity"][i]) < 1e-13


@pytest.mark.parametrize("k", [2, 3, 12, 17])
def test_apply_gate_all_positions_vs_oracle(k):
    rng = np.random.default_rng(k)
    psi = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    pairs = [(0, 1), (k - 2, k - 1), (k - 1, 0), (0, k - 1)]
    if k > 3:
        pairs += [(1, k - 2), (k // 2, 1), (k - 1, k // 2)]
    for t in pairs:
        g = manifold.random_unitary(4, rng)
        want = O.apply_gate(psi, g, t)
        assert rel_err(K.apply_gate(psi, K.Gate(g, t)), want) < 1e-14
        p = manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng))
        assert rel_err(K.apply_gate(psi, K.Gate(p, t)), O.apply_gate(psi, p, t)) < 1e-14
        bra = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
        assert rel_err(K.hole_contract(bra, psi, t), O.hole_contract(bra, psi, t)) < 1e-12


def test_apply_gate_errors():
    psi = np.ones(4, complex)
    with pytest.raises(ValueError):
        K.apply_gate(psi, K.Gate(np.eye(4), (0, 2)))
    with pytest.raises(ValueError):
        K.Gate(np.eye(4), (1, 1))
    with pytest.raises(ValueError):
        K.apply_gate(psi, K.Gate(np.eye(4), (0, 1)), out=psi)
    with pytest.raises(ValueError):
        K.apply_gate(np.ones(6, complex), K.Gate(np.eye(4), (0, 1)))


def test_large_vector_round_trip_and_norm():
    """Size-independent properties at 2^28 amplitudes (4 GiB): G then G^dag is
    the identity and the norm is preserved, for low / high / split targets."""
    k = 28
    rng = np.random.default_rng(1)
    dev = torch.device("cuda")
    x = torch.randn(2**k, dtype=torch.complex128, device=dev)
    x /= torch.linalg.vector_norm(x)
    y = x.clone()
    for t in [(0, 1), (26, 27), (27, 3), (5, 20)]:
        g = manifold.random_unitary(4, rng)
        y = K.apply_gate(y, K.Gate(g, t))
        n = torch.linalg.vector_norm(y).item()
        assert abs(n - 1.0) < 1e-12
        y = K.apply_gate(y, K.Gate(g.conj().T, t))
    assert torch.max(torch.abs(y - x)).item() < 1e-14 * 2 ** (k / 2) + 1e-12


# ------------------------------------------------------------ sector maps


def test_sector_maps_bit_exact():
    dev = torch.device("cuda")
    for sector in (0, 1):
        i = torch.arange(2**22, dtype=torch.int64, device=dev)
        x = torch.empty_like(i)
        gf._lib.check(gf._lib.lib.gf_sector_unrank(i.data_ptr(), i.numel(), sector, x.data_ptr(),
                                                   gf._lib.stream_ptr()))
        want = O.sector_unrank(i.cpu().numpy(), sector)
        assert np.array_equal(x.cpu().numpy(), want)
        back = torch.empty_like(i)
        gf._lib.check(gf._lib.lib.gf_sector_rank(x.data_ptr(), x.numel(), back.data_ptr(), gf._lib.stream_ptr()))
        assert torch.equal(back, i)
    # 2^31-entry sector of k = 32: spot check the top of the range
    i = torch.arange(2**31 - 4096, 2**31, dtype=torch.int64, device=dev)
    x = torch.empty_like(i)
    gf._lib.check(gf._lib.lib.gf_sector_unrank(i.data_ptr(), i.numel(), 0, x.data_ptr(), gf._lib.stream_ptr()))
    assert np.array_equal(x.cpu().numpy(), O.sector_unrank(i.cpu().numpy(), 0))


@pytest.mark.parametrize("L", [4, 6, 8])
def test_orbit_canon_bit_exact(L):
    dev = torch.device("cuda")
    rng = np.random.default_rng(L)
    x = rng.integers(0, 2 ** (2 * L), size=20000, dtype=np.int64)
    xd = torch.from_numpy(x).to(dev)
    rep, size = torch.empty_like(xd), torch.empty_like(xd)
    gf._lib.check(gf._lib.lib.gf_orbit_canon(xd.data_ptr(), xd.numel(), L, rep.data_ptr(), size.data_ptr(),
                                             gf._lib.stream_ptr()))
    r2, s2 = O.orbit_canon(x, L)
    assert np.array_equal(rep.cpu().numpy(), r2) and np.array_equal(size.cpu().numpy(), s2)


def test_fold_basis_matches_oracle_and_burnside():
    from paper_2506_23775_b200.objective import fold_basis

    for L in (4, 6):
        spec = fold_basis(2 * L, 0)
        reps, w = O.sector_orbit_reps(L, 0)
        assert np.array_equal(spec.indices, reps) and np.array_equal(spec.weights, w)
    assert fold_basis(8, 0).total == 72


def test_c1q_sector_gate_matches_full_space():
    rng = np.random.default_rng(3)
    k = 8
    for sector in (0, 1):
        full = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
        par = np.array([bin(j).count("1") & 1 for j in range(2**k)])
        full[par != sector] = 0
        sel = O.sector_unrank(np.arange(2 ** (k - 1)), sector)
        for a in (0, 3, 6):
            p = manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng))
            want = O.apply_gate(full, p, (a, k - 1))[sel]
            got = K.apply_sector_c1q(full[sel], p, a, k, sector)
            assert rel_err(got, want) < 1e-14
            # the swapped orientation (k-1, a) through the engine's wire swap
            want2 = O.apply_gate(full, p, (k - 1, a))[sel]
            got2 = K.apply_sector_c1q(full[sel], K.wire_swapped_matrix(p), a, k, sector)
            assert rel_err(got2, want2) < 1e-14


@pytest.mark.parametrize("k", [1, 2, 5, 17])
def test_apply_gate_1q_every_qubit_vs_oracle(k):
    """Generic one-qubit gate on every qubit against the oracle's restatement
    of reference apply_gate with kron(g, I) (the reference embeds 1q gates in
    its 2q gates), and batched / in-place through the ABI."""
    rng = np.random.default_rng(40 + k)
    psi = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
    for q in range(k):
        g = manifold.random_unitary(2, rng)
        got = K.apply_gate_1q(psi, g, q)
        if k == 1:
            want = g @ psi
        else:
            other = q + 1 if q + 1 < k else q - 1
            pair = (q, other)
            want = O.apply_gate(psi, np.kron(g, np.eye(2)), pair)
        assert rel_err(got, want) < 1e-14
    # batched, in place, on the device
    x = torch.from_numpy(np.stack([psi, 2 * psi])).cuda()
    g = manifold.random_unitary(2, rng)
    gg = np.ascontiguousarray(g)
    gf._lib.check(gf._lib.lib.gf_apply_gate_1q(x.data_ptr(), x.data_ptr(), k, 0, gg.ctypes.data, 2,
                                               gf._lib.stream_ptr()))
    want = K.apply_gate_1q(psi, g, 0)
    assert rel_err(x[1].cpu().numpy(), 2 * want) < 1e-14 and rel_err(x[0].cpu().numpy(), want) < 1e-14
    with pytest.raises(ValueError):
        K.apply_gate_1q(psi, g, k)
    with pytest.raises(ValueError):
        K.apply_gate_1q(psi, np.eye(4), 0)


def test_apply_gate_on_16_byte_aligned_views():
    """K1 moves aligned amplitude pairs with 256-bit accesses; a tensor view at
    an odd amplitude offset (16 B aligned only) must take the 128-bit path and
    give the same result as an aligned copy (no misaligned-address fault)."""
    import torch

    rng = np.random.default_rng(5)
    k = 10
    st = gf._lib.stream_ptr()
    for t in [(k - 2, k - 1), (3, k - 1), (1, 2), (0, 5)]:
        g = np.ascontiguousarray(manifold.random_unitary(4, rng))
        host = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
        buf = torch.zeros(2**k + 1, dtype=torch.complex128, device="cuda")
        view = buf[1:]
        view.copy_(torch.from_numpy(host))
        assert view.data_ptr() % 32 == 16
        gf._lib.check(gf._lib.lib.gf_apply_gate(view.data_ptr(), view.data_ptr(), k, t[0], t[1], g.ctypes.data, 0, 1,
                                                st))
        assert rel_err(view.cpu().numpy(), O.apply_gate(host, g, t)) < 1e-14
    p = np.ascontiguousarray(manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng)))
    for a in (0, 4, k - 2):
        full = rng.normal(size=2**k) + 1j * rng.normal(size=2**k)
        par = np.array([bin(j).count("1") & 1 for j in range(2**k)])
        full[par != 0] = 0
        sel = O.sector_unrank(np.arange(2 ** (k - 1)), 0)
        buf = torch.zeros(2 ** (k - 1) + 1, dtype=torch.complex128, device="cuda")
        view = buf[1:]
        view.copy_(torch.from_numpy(full[sel]))
        gf._lib.check(gf._lib.lib.gf_apply_gate_sector_c1q(view.data_ptr(), view.data_ptr(), k, a, 0, p.ctypes.data, 1,
                                                           st))
        assert rel_err(view.cpu().numpy(), O.apply_gate(full, p, (a, k - 1))[sel]) < 1e-14


# ------------------------------------------------------------------ engine


def _c1():
    g = golden("c1")
    spec, circ, rng = gf.spinful_layer_circuit(4, 3, False, seed=0)
    assert np.array_equal(circ.gate_stack(), g["gates"])
    orc = gf.DenseOracle(spec, 0.25)
    return g, spec, circ, orc


def test_c1_dense_target_on_gpu_matches_reference():
    g, spec, circ, orc = _c1()
    assert rel_err(orc._u[:, :4], g["U_cols"]) < 1e-12


def test_c1_value_gradient_hvp_vs_reference():
    g, spec, circ, orc = _c1()
    X = list(g["direction"])
    assert abs(gf.target_value(circ, orc) - g["target_value"]) < TOL * abs(g["target_value"])
    rep = gf.full_gradient(circ, orc)
    assert abs(rep.value - g["value"]) < TOL * abs(g["value"])
    assert rel_err(np.stack(rep.holomorphic_derivatives), g["holo"]) < TOL
    assert rel_err(np.stack(rep.per_logical_gradient), g["riem"]) < TOL
    assert [rep.pass_counts[n] for n in gf.objective.COUNT_NAMES] == list(g["grad_counts"])
    hv = gf.hessian_vector_product(circ, orc, X)
    assert rel_err(np.stack(hv), g["hvp"]) < TOL
    rep2, hv2 = gf.gradient_and_hvp(circ, orc, X)
    assert rel_err(np.stack(hv2), g["hvp"]) < TOL
    assert rel_err(np.stack(rep2.holomorphic_derivatives), g["holo"]) < TOL
    hx = [manifold.hessian_apply_gate(gg.matrix, e, manifold.euclid_gradient_from_holomorphic(h), x)
          for gg, e, h, x in zip(circ.logical_gates, rep.euclidean_gradients, hv, X)]
    assert abs(sum(manifold.inner(x, y) for x, y in zip(X, hx)) - g["x_hess_x"]) < TOL * abs(g["x_hess_x"])


def test_c1_full_hessian_vs_reference():
    g, spec, circ, orc = _c1()
    rep = gf.full_hessian(circ, orc)
    keys = [tuple(int(v) for v in x) for x in g["hess_keys"]]
    assert sorted(rep.hessian.blocks) == keys
    scale = np.abs(g["hess_blocks"]).max()
    for kk, ref in zip(keys, g["hess_blocks"]):
        assert np.abs(rep.hessian.blocks[kk] - ref).max() < TOL * scale
    assert [rep.pass_counts[n] for n in gf.objective.COUNT_NAMES] == list(g["hess_counts"])


def test_c1_full_hessian_pair_csr_driver_vs_reference():
    """The reference's own Hessian algorithm on the GPU (gf_hess_plan_eval:
    cached passes, hole arrays, routed pair contractions): blocks, value,
    gradient and every pass counter equal the reference's c1 run, for
    several batch / chunk shapes (bit-identical records across them)."""
    g, spec, circ, orc = _c1()
    keys = [tuple(x) for x in g["hess_keys"]]
    ref = None
    for batch, chunk in ((256, 64), (64, 64), (32, 16)):
        rep = gf.full_hessian(circ, orc, method="pairs", batch=batch, chunk=chunk)
        assert rep.engine["hessian_method"] == "pairs"
        assert sorted(rep.hessian.blocks) == keys
        for kk, b in zip(keys, g["hess_blocks"]):
            assert rel_err(rep.hessian.blocks[kk], b) < TOL
        assert abs(rep.value - g["value"]) < TOL * abs(g["value"])
        assert rel_err(np.stack(rep.holomorphic_derivatives), g["holo"]) < TOL
        assert [rep.pass_counts[c] for c in gf.objective.COUNT_NAMES] == [int(x) for x in g["hess_counts"]]
        if chunk == 64:
            if ref is None:
                ref = rep
            else:
                for kk in keys:
                    assert np.array_equal(rep.hessian.blocks[kk], ref.hessian.blocks[kk])


def test_c1_trust_region_five_iterations_vs_reference():
    g, spec, circ, orc = _c1()
    final, trace = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=5))
    f = np.array([r.value for r in trace.records])
    assert np.allclose(f, g["tr_f"], rtol=1e-9, atol=1e-9)
    assert [r.accepted for r in trace.records] == list(g["tr_accepted"])
    assert [r.stop_reason for r in trace.records] == list(g["tr_reason"])
    assert np.allclose([r.radius for r in trace.records], g["tr_radius"], rtol=1e-9)
    assert rel_err(np.stack([x.matrix for x in final.logical_gates]), g["tr_final_gates"]) < 1e-8


def test_batch_and_chunk_bit_determinism():
    g, spec, circ, orc = _c1()
    X = list(g["direction"])
    base = gf.gradient_and_hvp(circ, orc, X, batch=256)
    for b in (64, 128):
        other = gf.gradient_and_hvp(circ, orc, X, batch=b)
        assert other[0].value == base[0].value
        assert np.array_equal(np.stack(other[0].holomorphic_derivatives), np.stack(base[0].holomorphic_derivatives))
        assert np.array_equal(np.stack(other[1]), np.stack(base[1]))


def test_random_circuit_matrix_oracle_and_shared_gates():
    """Random wire pairs (adjacent / general / swapped) with a Haar target."""
    rng = np.random.default_rng(9)
    k = 7
    u = manifold.random_unitary(2**k, rng)
    gates, slots = [], []
    for i in range(9):
        t1, t2 = (int(x) for x in rng.choice(k, size=2, replace=False))
        gates.append(gf.Gate(manifold.random_unitary(4, rng), (t1, t2)))
        slots.append(gf.GateSlot(i % 5, (t1, t2)))
    circ = gf.Circuit(k, slots, gates[:5])
    orc = gf.DenseOracle.from_matrix(u)
    X = [rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)) for _ in range(5)]
    rep, hv = gf.gradient_and_hvp(circ, orc, X)
    t1, t2, lid = circ.slot_arrays()
    plan = O.Plan(k, np.stack([t1, t2], 1), lid, circ.gate_stack())
    phi = O.dense_phi0(u)
    v, d, _ = O.gradient_sum(plan, np.arange(2**k), phi)
    h, _ = O.hvp_sum(plan, X, np.arange(2**k), phi)
    assert abs(rep.value + v.real) < TOL * max(1, abs(v))
    assert rel_err(np.stack(rep.holomorphic_derivatives), plan.logical_sum(d)) < TOL
    assert rel_err(np.stack(hv), plan.logical_sum(h)) < TOL


def test_empty_circuit_and_oracle_mismatch():
    circ = gf.Circuit(4, [], [])
    orc = gf.DenseOracle.from_matrix(np.eye(16, dtype=complex))
    assert gf.target_value(circ, orc) == -16.0
    with pytest.raises(ValueError):
        gf.target_value(gf.Circuit(3, [], []), orc)


@pytest.mark.parametrize("name", ["sector_l4p", "sector_l6p", "sector_l5o"])
def test_sector_engine_vs_reference_restricted_sums(name):
    g = golden(name)
    k, L = int(g["k"]), int(g["L"])
    spec, circ, rng = gf.spinful_layer_circuit(L, int(g["gates"].shape[0]), bool(g["periodic"]),
                                               seed={"sector_l4p": 2, "sector_l6p": 4, "sector_l5o": 5}[name],
                                               parity=True)
    assert np.array_equal(circ.gate_stack(), g["gates"])
    orc = gf.DenseOracle(spec, 0.25)
    X = list(g["direction"])
    for sect, nm in ((0, "even"), (1, "odd")):
        rep, hv = gf.gradient_and_hvp(circ, orc, X, parity_mode=True, sector=sect)
        ref_v = g[nm + "_value"]
        assert abs(-rep.value - ref_v.real) < TOL * max(1, abs(ref_v))
        assert rel_err(np.stack(rep.holomorphic_derivatives), g[nm + "_holo"]) < TOL
        assert rel_err(np.stack(hv), g[nm + "_hvp"]) < TOL


@pytest.mark.parametrize("knobs", [{"GF_SECTOR_FMA": "0"}, {"GF_UNIT_NT": "128"}, {"GF_FUSED_M": "8"},
                                   {"GF_FUSED_M": "9", "GF_UNIT_NT": "128"}, {"GF_FUSED_M": "6"}])
def test_sector_engine_variants_vs_reference_sums(monkeypatch, knobs):
    """The parity-sector passes run as FP64-FMA units (PM_UNIT) by default.
    The other builds of the same sweeps -- the DMMA sector path
    (GF_SECTOR_FMA=0: structural-zero parity gates, PM_C1QD slots), 128-thread
    unit CTAs, forced small tiles (several tiles and passes; 2^6 tiles fall
    back to the DMMA path) -- must reproduce the reference-derived sector sums."""
    for k_, v_ in knobs.items():
        monkeypatch.setenv(k_, v_)
    g = golden("sector_l6p")
    L = int(g["L"])
    spec, circ, rng = gf.spinful_layer_circuit(L, int(g["gates"].shape[0]), bool(g["periodic"]), seed=4, parity=True)
    orc = gf.DenseOracle(spec, 0.25)
    X = list(g["direction"])
    for sect, nm in ((0, "even"), (1, "odd")):
        rep, hv = gf.gradient_and_hvp(circ, orc, X, parity_mode=True, sector=sect)
        ref_v = g[nm + "_value"]
        assert abs(-rep.value - ref_v.real) < TOL * max(1, abs(ref_v))
        assert rel_err(np.stack(rep.holomorphic_derivatives), g[nm + "_holo"]) < TOL
        assert rel_err(np.stack(hv), g[nm + "_hvp"]) < TOL
        grad = gf.full_gradient(circ, orc, parity_mode=True, sector=sect)  # OP_REV_G passes
        assert rel_err(np.stack(grad.holomorphic_derivatives), g[nm + "_holo"]) < TOL
        hv1 = gf.hessian_vector_product(circ, orc, X, sector=sect)          # OP_REV_H passes
        assert rel_err(np.stack(hv1), g[nm + "_hvp"]) < TOL
        val = gf.target_value(circ, orc, sector=sect)                        # OP_FWD_DOT
        assert abs(-val - ref_v.real) < TOL * max(1, abs(ref_v))


@pytest.mark.parametrize("case", ["c2_slice", "sector"])
def test_light_cone_rule_changes_nothing(monkeypatch, case):
    """Dead-tile skipping (tiles outside the basis state's light cone hold
    psi = v = 0 and are skipped in the reverse and ascending sweeps alike) is
    exact: value, gradient and HVP agree with GF_LIGHTCONE=0 to rounding, and
    the plan reports how much slot work is left."""
    from paper_2506_23775_b200 import objective as obj

    if case == "c2_slice":
        spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
        orc = gf.ChebyshevOracle(spec, 0.25)
        kw = dict(basis=np.arange(96, dtype=np.int64) * 677 % 65536)
        parity = False
    else:
        spec, circ, rng = gf.spinful_layer_circuit(7, 4, True, seed=11, parity=True)
        orc = gf.ChebyshevOracle(spec, 0.25)
        kw = dict(sector=0, basis=(np.arange(40, dtype=np.int64) * 211 % (1 << 13), None))
        parity = True
    X = [manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
         for g in circ.logical_gates]
    out = {}
    for lc in ("1", "0"):
        monkeypatch.setenv("GF_LIGHTCONE", lc)
        rep, hv = gf.gradient_and_hvp(circ, orc, X, parity_mode=parity, **kw)
        live = list(obj._PLANS.values())[-1].describe()["live_fraction"]
        out[lc] = (rep.value, np.stack(rep.holomorphic_derivatives), np.stack(hv), live)
    assert abs(out["1"][0] - out["0"][0]) < 1e-12 * max(1.0, abs(out["0"][0]))
    assert rel_err(out["1"][1], out["0"][1]) < 1e-12
    assert rel_err(out["1"][2], out["0"][2]) < 1e-12
    assert all(v == 1.0 for v in out["0"][3].values())
    assert all(0.0 < v <= 1.0 for v in out["1"][3].values()) and out["1"][3]["forward"] < 1.0
    assert out["1"][3]["reverse"] == out["1"][3]["ascending"]


@pytest.mark.parametrize("name", ["sector_l4p", "sector_l6p"])
def test_fold_engine_vs_reference_even_sum(name):
    g = golden(name)
    L = int(g["L"])
    spec, circ, rng = gf.spinful_layer_circuit(L, 3, True, seed={"sector_l4p": 2, "sector_l6p": 4}[name],
                                               parity=True)
    orc = gf.DenseOracle(spec, 0.25)
    X = list(g["direction"])
    rep, hv = gf.gradient_and_hvp(circ, orc, X, parity_mode=True, sector="even", fold=True)
    assert abs(-rep.value - g["even_value"].real) < TOL * max(1, abs(g["even_value"]))
    assert rel_err(np.stack(rep.holomorphic_derivatives), g["even_holo"]) < TOL
    assert rel_err(np.stack(hv), g["even_hvp"]) < TOL


def test_chebyshev_oracle_matches_dense_and_reference_krylov():
    g = golden("models")
    spec = gf.build_spinful_fh(3, 1.0, 4.0, True)
    orc = gf.ChebyshevOracle(spec, 0.25)
    assert rel_err(orc.apply(g["krylov_in"]), g["dense_out"]) < 1e-12
    spec4 = gf.build_spinful_fh(4, 1.0, 4.0, False)
    d = gf.DenseOracle(spec4, 0.25)
    c = gf.ChebyshevOracle(spec4, 0.25)
    js = torch.arange(0, 256, dtype=torch.int64, device="cuda")
    a = torch.empty((256, 256), dtype=torch.complex128, device="cuda")
    b = torch.empty_like(a)
    d.phi0_into(js, None, a)
    c.phi0_into(js, None, b)
    assert torch.max(torch.abs(a - b)).item() < 1e-13



@pytest.mark.parametrize("mode", ["tables", "blocks", "columns"])
def test_number_block_oracle_matches_dense(mode):
    """Block-coordinate Chebyshev (colex ranks, O(1) adjacent-hop rank steps,
    periodic wrap bonds by full re-rank) == dense expm, full and sector rows,
    whole-block cache and per-column modes."""
    for spec in (gf.build_spinful_fh(4, 1.0, 4.0, False), gf.build_spinful_fh(3, 0.7, 2.5, True),
                 gf.build_spinless_fh(7, 1.0, 3.0, True)):
        k = spec.num_qubits
        d = gf.DenseOracle(spec, 0.25)
        nb = gf.NumberBlockOracle(spec, 0.25, cache_dim=0 if mode == "columns" else 8192)
        if mode == "blocks":
            nb._tab = False  # per-group path with cached block matrices
        js = torch.arange(0, 1 << k, dtype=torch.int64, device="cuda")
        a = torch.empty((1 << k, 1 << k), dtype=torch.complex128, device="cuda")
        b = torch.full_like(a, 7.0)
        d.phi0_into(js, None, a)
        nb.phi0_into(js, None, b)
        assert torch.max(torch.abs(a - b)).item() < 1e-13
        for sector in (0, 1):
            st = torch.arange(0, 1 << (k - 1), dtype=torch.int64, device="cuda")
            jf = torch.from_numpy(O.sector_unrank(st.cpu().numpy(), sector)).cuda()
            a2 = torch.empty((1 << (k - 1), 1 << (k - 1)), dtype=torch.complex128, device="cuda")
            b2 = torch.full_like(a2, 7.0)
            d.phi0_into(jf, sector, a2)
            nb.phi0_into(jf, sector, b2)
            assert torch.max(torch.abs(a2 - b2)).item() < 1e-13


def test_number_block_oracle_c2_reference_krylov_checks():
    """configs[1] target columns from the number-block oracle against the
    reference Krylov phi0 checksums (tests/golden/c2_slice.npz), then the
    c2 slice gradient / HVP through it."""
    g = golden("c2_slice")
    spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
    orc = gf.NumberBlockOracle(spec, 0.25)
    js = g["js"]
    srng = np.random.default_rng(2)
    srng.choice(2**16, size=16, replace=False)
    w = srng.normal(size=2**16) + 1j * srng.normal(size=2**16)
    phi = torch.empty((16, 2**16), dtype=torch.complex128, device="cuda")
    orc.phi0_into(torch.from_numpy(js).cuda(), None, phi)
    P = phi.cpu().numpy()
    chk = np.array([[p.sum(), p @ w, np.vdot(p, p).real] for p in P])
    assert rel_err(chk, g["phi_checks"]) < 1e-10
    rep, hv = gf.gradient_and_hvp(circ, orc, list(g["direction"]), basis=js)
    assert rel_err(np.stack(rep.holomorphic_derivatives), g["holo"]) < TOL
    assert rel_err(np.stack(hv), g["hvp"]) < TOL

def test_c2_slice_vs_reference_chunk_drivers():
    """BASELINE configs[1] (16 qubits, 36 slots): reference _gradient_chunk /
    _hvp_chunk with Krylov phi0 on a seeded 16-state sample."""
    g = golden("c2_slice")
    spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
    assert np.array_equal(circ.gate_stack(), g["gates"])
    orc = gf.ChebyshevOracle(spec, 0.25)
    js = g["js"]
    srng = np.random.default_rng(2)
    srng.choice(2**16, size=16, replace=False)
    w = srng.normal(size=2**16) + 1j * srng.normal(size=2**16)
    phi = torch.empty((16, 2**16), dtype=torch.complex128, device="cuda")
    orc.phi0_into(torch.from_numpy(js).cuda(), None, phi)
    P = phi.cpu().numpy()
    chk = np.array([[p.sum(), p @ w, np.vdot(p, p).real] for p in P])
    assert rel_err(chk, g["phi_checks"]) < 1e-10
    rep, hv = gf.gradient_and_hvp(circ, orc, list(g["direction"]), basis=js)
    assert abs(-rep.value - g["values"].sum().real) < TOL * max(1, abs(g["values"].sum()))
    assert rel_err(np.stack(rep.holomorphic_derivatives), g["holo"]) < TOL
    assert rel_err(np.stack(hv), g["hvp"]) < TOL


def test_k20_single_summands_vs_oracle():
    """Larger vectors (2^20 amplitudes; multi-CTA reductions per summand)."""
    spec, circ, rng = gf.spinful_layer_circuit(10, 4, False, seed=3)
    X = [manifold.project_tangent_gate(x.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))
         for x in circ.logical_gates]
    orc = gf.ChebyshevOracle(spec, 0.25)
    js = np.array([5, 77777, 1000001])
    rep, hv = gf.gradient_and_hvp(circ, orc, X, basis=js)
    phi = torch.empty((3, 2**20), dtype=torch.complex128, device="cuda")
    orc.phi0_into(torch.from_numpy(js).cuda(), None, phi)
    P = phi.cpu().numpy()
    t1, t2, lid = circ.slot_arrays()
    plan = O.Plan(20, np.stack([t1, t2], 1), lid, circ.gate_stack())
    fn = lambda jj: P[np.searchsorted(js, jj)]
    v, d, _ = O.gradient_sum(plan, js, fn)
    h, _ = O.hvp_sum(plan, X, js, fn)
    assert abs(rep.value + v.real) < TOL * max(1, abs(v))
    assert rel_err(np.stack(rep.holomorphic_derivatives), plan.logical_sum(d)) < TOL
    assert rel_err(np.stack(hv), plan.logical_sum(h)) < TOL


@pytest.mark.parametrize("engine,m", [("fused", "6"), ("fused", "7"), ("fused", "12"), ("stream", None)])
def test_multi_tile_multi_pass_engine_vs_oracle(monkeypatch, engine, m):
    """Force tiny fused tiles (2^6 amplitudes) on a 12-qubit circuit: many
    tiles per vector and many passes per sweep, both sector and full space."""
    monkeypatch.setenv("GF_ENGINE", engine)
    if m:
        monkeypatch.setenv("GF_FUSED_M", m)
    for sector, parity in ((None, False), (0, True)):
        spec, circ, rng = gf.spinful_layer_circuit(6, 5, True, seed=12, parity=parity)
        X = [manifold.project_tangent_gate(x.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
             for x in circ.logical_gates]
        orc = gf.DenseOracle(spec, 0.25)
        rep, hv = gf.gradient_and_hvp(circ, orc, X, parity_mode=parity, sector=sector, batch=64)
        t1, t2, lid = circ.slot_arrays()
        plan = O.Plan(12, np.stack([t1, t2], 1), lid, circ.gate_stack())
        js = np.arange(4096) if sector is None else np.sort(O.sector_unrank(np.arange(2048), 0))
        phi = O.dense_phi0(orc._u)
        v, d, _ = O.gradient_sum(plan, js, phi, workers=8)
        h, _ = O.hvp_sum(plan, X, js, phi, workers=8)
        hol, hvo = plan.logical_sum(d), plan.logical_sum(h)
        if sector is not None:
            mask = np.array([[(i ^ (i >> 1)) & 1 == (j ^ (j >> 1)) & 1 for j in range(4)] for i in range(4)])
            hol, hvo = hol * mask, hvo * mask
        assert abs(rep.value + v.real) < TOL * max(1, abs(v))
        assert rel_err(np.stack(rep.holomorphic_derivatives), hol) < TOL
        assert rel_err(np.stack(hv), hvo) < TOL


def test_integration_stub_matches_reference_chunk_drivers():
    """pure-ctypes stub (gf_malloc / gf_memcpy /
    gf_plan_eval / gf_plan_slot_outputs) returns the reference drivers'
    per-slot dacc / oacc for a chunk."""
    import integration_stub as S

    g = golden("c1")
    spec, circ, rng = gf.spinful_layer_circuit(4, 3, False, seed=0)
    orc = gf.DenseOracle(spec, 0.25)
    ev = S.GpuChunkEvaluator(circ, max_chunk=64)
    ev.set_directions(g["direction"])
    t1, t2, lid = circ.slot_arrays()
    plan = O.Plan(8, np.stack([t1, t2], 1), lid, circ.gate_stack())
    phi = O.dense_phi0(orc._u)
    vals, dsum, hsum = 0j, 0, 0
    for j0 in range(0, 256, 64):
        phi0s = phi(np.arange(j0, j0 + 64))
        v, dacc, oacc = ev(S.GF_VALUE | S.GF_GRAD | S.GF_HVP, j0, j0 + 64, phi0s)
        ov, od, _ = O.gradient_sum(plan, np.arange(j0, j0 + 64), phi)
        oh, _ = O.hvp_sum(plan, list(g["direction"]), np.arange(j0, j0 + 64), phi)
        assert abs(v - ov) < TOL * max(1, abs(ov))
        assert rel_err(dacc.reshape(-1, 16), od) < TOL
        assert rel_err(oacc.reshape(-1, 16), oh) < TOL
        vals += v
        dsum = dsum + dacc
    assert abs(-vals.real - g["value"]) < TOL * abs(g["value"])
    assert rel_err(plan.logical_sum(dsum.reshape(-1, 16)), g["holo"]) < TOL


def test_integration_stub_hessian_chunk_with_dedup_vs_reference():
    """INTEGRATION.md section B, Hessian: the ctypes stub's
    GpuHessianChunkEvaluator (gf_hess_plan_*) fed the reference's dedup pair
    CSR (translation classes from the reference fixture) returns the
    reference's blocks, dacc and counters for full_hessian's chunk closure
    (objective.py:729-744)."""
    import integration_stub as S

    g = golden("dedup")
    k = int(g["k"])
    circ = gf.Circuit(k, [gf.GateSlot(int(l), tuple(int(x) for x in t)) for t, l in zip(g["targets"], g["logical"])],
                      [gf.Gate(m, (0, 1)) for m in g["gates"]],
                      gf.BrickwallMeta(3, tuple(int(l) for l in g["logical"]), 2, True))
    classes = [((int(a), int(b)), int(m)) for a, b, m in g["classes"]]
    csr = O.pair_csr(g["targets"], g["logical"], len(g["gates"]), classes)
    ev = S.GpuHessianChunkEvaluator(circ, O.DENSE_SUPPORT, csr, max_chunk=64)
    phi = O.dense_phi0(g["U"])
    tot_v, tot_d, tot_b, tot_c = 0j, 0, 0, 0
    for j0 in range(0, 64, 32):
        v, dacc, blocks, counts = ev(j0, j0 + 32, phi(np.arange(j0, j0 + 32)))
        tot_v, tot_d, tot_b, tot_c = tot_v + v, tot_d + dacc, tot_b + blocks, tot_c + counts
    assert np.array_equal(tot_c, g["dedup_counts"])
    keys = [tuple(int(x) for x in kk) for kk in g["dedup_keys"]]
    nlog = len(g["gates"])
    sc = np.abs(g["dedup_blocks"]).max()
    for (a, b), ref in zip(keys, g["dedup_blocks"]):
        r = a * nlog - a * (a - 1) // 2 + (b - a)
        assert np.abs(tot_b[r] - ref).max() < TOL * sc
    t1, t2, lid = circ.slot_arrays()
    plan = O.Plan(k, np.stack([t1, t2], 1), lid, circ.gate_stack())
    assert rel_err(plan.logical_sum(tot_d.reshape(-1, 16)), g["holo"]) < TOL
    assert abs(-tot_v.real - g["value"]) < TOL * abs(g["value"])


@pytest.mark.parametrize("sector,m", [(None, None), (0, None), (None, "7")])
def test_multi_direction_hvp_equals_single(monkeypatch, sector, m):
    """gf_plan_set_directions_multi: 3 directions in one set of sweeps give the
    same HVPs as three separate evaluations (full space, sector with
    parity-controlled slots, forced small tiles)."""
    if m:
        monkeypatch.setenv("GF_FUSED_M", m)
    parity = sector is not None
    spec, circ, rng = gf.spinful_layer_circuit(5, 4, False, seed=21, parity=parity)
    orc = gf.DenseOracle(spec, 0.25)
    dirs = []
    for _ in range(3):
        dirs.append([manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)),
                                                   parity) for g in circ.logical_gates])
    dirs[2][1] = np.zeros((4, 4), complex)  # a zero logical block exercises the skipped Z-terms
    multi = gf.hessian_vector_products(circ, orc, dirs, sector=sector)
    for z, got in zip(dirs, multi):
        one = gf.hessian_vector_product(circ, orc, z, sector=sector)
        assert rel_err(np.stack(got), np.stack(one)) < 1e-12


def test_non_finite_engine_output_raises_floating_point_error():
    """GF_ENONFINITE: a NaN in a gate propagates into the records and is
    reported as FloatingPointError (reference objective.py:575-578), for the
    engine and the pair-CSR Hessian driver alike."""
    g, spec, circ, orc = _c1()
    bad = circ.gate_stack().copy()
    bad[1, 2, 3] = np.nan
    cb = circ.with_gates(list(bad))
    with pytest.raises(FloatingPointError):
        gf.full_gradient(cb, orc)
    with pytest.raises(FloatingPointError):
        gf.full_hessian(cb, orc, method="pairs")
    x = torch.tensor([1.0, np.inf, 0.0], dtype=torch.float64, device="cuda")
    with pytest.raises(FloatingPointError):
        gf._lib.check(gf._lib.lib.gf_check_finite(x.data_ptr(), 3, gf._lib.stream_ptr()))
    gf._lib.check(gf._lib.lib.gf_check_finite(x.data_ptr(), 1, gf._lib.stream_ptr()))
