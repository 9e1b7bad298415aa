"""Pin the CPU oracle (oracle/) against fixtures from the unmodified reference.

Every check here compares oracle output with tests/golden/*.npz produced by
tests/golden/make_golden.py running gatefit itself.  No GPU needed.
"""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import gf_oracle as O


def test_kernels_match_reference_vectors():
    g = golden("kernels")
    psi, bra = g["psi"], g["bra"]
    for i, t in enumerate(g["pairs"]):
        t = tuple(int(x) for x in t)
        t2 = tuple(int(x) for x in g["second_pairs"][i])
        assert rel_err(O.apply_gate(psi, g["gates"][i], t), g["apply"][i]) < 1e-14
        assert rel_err(O.apply_gate(psi, g["pgates"][i], t, sparse=True), g["apply_parity"][i]) < 1e-14
        assert rel_err(O.hole_contract(bra, psi, t), g["hole_contract"][i]) < 1e-14
        arr = O.hole_apply(psi, t)
        assert np.array_equal(arr, g["hole_apply"][i])
        arrp = O.hole_apply(psi, t, O.PARITY_SUPPORT)
        assert np.array_equal(arrp, g["hole_apply_parity"][i])
        assert rel_err(O.apply_gate_to_array(arr, g["gates"][i], t2), g["array_apply"][i]) < 1e-14
        assert rel_err(O.hole_contract_array(bra, arr, t2), g["hole_contract_array"][i]) < 1e-14
        assert rel_err(O.hole_contract_array(bra, arrp, t2, O.PARITY_SUPPORT),
                       g["hole_contract_array_parity"][i]) < 1e-14


def _c1():
    g = golden("c1")
    terms, groups = O.spinful_terms(4, 1.0, 4.0, False)
    U = O.dense_target(8, terms, 0.25)
    return g, U


def test_c1_dense_target_matches_reference():
    g, U = _c1()
    assert rel_err(U[:, :4], g["U_cols"]) < 1e-12
    assert rel_err(np.diag(U), g["U_diag"]) < 1e-12


def test_c1_value_gradient_hvp_hessian():
    g, U = _c1()
    k = int(g["k"])
    plan = O.Plan(k, g["targets"], g["logical"], g["gates"])
    js = np.arange(2**k)
    phi = O.dense_phi0(U)
    v, d, counts = O.gradient_sum(plan, js, phi, workers=4)
    assert abs(-v.real - g["value"]) < 1e-12 * abs(g["value"])
    holo = plan.logical_sum(d)
    assert rel_err(holo, g["holo"]) < 1e-12
    assert np.array_equal(counts, g["grad_counts"])
    vv, _ = O.value_sum(plan, js, phi)
    assert abs(-vv.real - g["target_value"]) < 1e-12
    h, _ = O.hvp_sum(plan, list(g["direction"]), js, phi, workers=4)
    assert rel_err(plan.logical_sum(h), g["hvp"]) < 1e-12
    vh, dh, blocks, hc = O.hessian_sum(plan, js, phi, workers=4)
    keys = [tuple(x) for x in g["hess_keys"]]
    assert sorted(blocks) == keys
    for kk, ref in zip(keys, g["hess_blocks"]):
        assert rel_err(blocks[kk], ref) < 1e-12
    assert np.array_equal(hc, g["hess_counts"])


def test_worker_count_bit_determinism():
    g, U = _c1()
    plan = O.Plan(8, g["targets"], g["logical"], g["gates"])
    js = np.arange(256)
    phi = O.dense_phi0(U)
    ref = O.gradient_sum(plan, js, phi, workers=1)
    for w in (2, 4, 8):
        got = O.gradient_sum(plan, js, phi, workers=w)
        assert got[0] == ref[0] and np.array_equal(got[1], ref[1])


@pytest.mark.parametrize("name", ["sector_l4p", "sector_l6p", "sector_l5o"])
def test_sector_restricted_sums(name):
    g = golden(name)
    k = int(g["k"])
    L = int(g["L"])
    terms, _ = O.spinful_terms(L, 1.0, 4.0, bool(g["periodic"]))
    U = O.dense_target(k, terms, 0.25)
    phi = O.dense_phi0(U)
    plan = O.Plan(k, g["targets"], g["logical"], g["gates"], parity_mode=True)
    hplan = O.Plan(k, g["targets"], g["logical"], g["gates"], parity_mode=False)
    X = list(g["direction"])
    for sect, nm in ((0, "even"), (1, "odd")):
        js = O.sector_unrank(np.arange(2 ** (k - 1)), sect)
        js.sort()
        v, d, _ = O.gradient_sum(plan, js, phi, workers=4)
        assert abs(v - g[nm + "_value"]) < 1e-12 * max(1, abs(g[nm + "_value"]))
        assert rel_err(plan.logical_sum(d), g[nm + "_holo"]) < 1e-11
        h, _ = O.hvp_sum(hplan, X, js, phi, workers=4)
        assert rel_err(hplan.logical_sum(h), g[nm + "_hvp"]) < 1e-11
    # even + odd = full trace
    assert abs(-(g["even_value"] + g["odd_value"]).real - g["full_value"]) < 1e-11 * (2**k)


@pytest.mark.parametrize("name", ["sector_l4p", "sector_l6p"])
def test_translation_fold_matches_even_sector_sum(name):
    g = golden(name)
    k = int(g["k"])
    L = int(g["L"])
    terms, _ = O.spinful_terms(L, 1.0, 4.0, True)
    U = O.dense_target(k, terms, 0.25)
    reps, w = O.sector_orbit_reps(L, 0)
    assert int(w.sum()) == 2 ** (k - 1)
    js = O.sector_unrank(reps, 0)
    Uc = np.conj(U).T
    phi = lambda jj: Uc[np.asarray(jj)] * w[np.searchsorted(js, jj)][:, None]
    plan = O.Plan(k, g["targets"], g["logical"], g["gates"], parity_mode=True)
    v, d, _ = O.gradient_sum(plan, js, phi)
    assert abs(v - g["even_value"]) < 1e-12 * max(1, abs(g["even_value"]))
    assert rel_err(plan.logical_sum(d), g["even_holo"]) < 1e-11


def test_burnside_orbit_count_l4():
    reps, w = O.sector_orbit_reps(4, 0)
    assert len(reps) == 72


def test_rank_unrank_bijection_exhaustive():
    for k in range(2, 17):
        M = 2 ** (k - 1)
        for sect in (0, 1):
            x = O.sector_unrank(np.arange(M), sect)
            par = np.array([bin(int(v)).count("1") & 1 for v in x[: min(M, 4096)]])
            assert np.all(par == sect)
            assert np.array_equal(O.sector_rank(x), np.arange(M))
            assert len(np.unique(x)) == M and x.max() < 2**k


def test_dedup_hessian_matches_reference():
    g = golden("dedup")
    plan = O.Plan(int(g["k"]), g["targets"], g["logical"], g["gates"])
    phi = O.dense_phi0(g["U"])
    js = np.arange(2 ** int(g["k"]))
    classes = [((int(a), int(b)), int(m)) for a, b, m in g["classes"]]
    for tag, cl in (("full_", None), ("dedup_", classes)):
        v, d, blocks, counts = O.hessian_sum(plan, js, phi, classes=cl, workers=4)
        keys = [tuple(x) for x in g[tag + "keys"]]
        assert sorted(blocks) == keys
        for kk, ref in zip(keys, g[tag + "blocks"]):
            assert rel_err(blocks[kk], ref) < 1e-12
        assert np.array_equal(counts, g[tag + "counts"])


def test_parity_mode_hessian_matches_reference():
    g = golden("dedup")
    plan = O.Plan(int(g["p_k"]), g["p_targets"], g["p_logical"], g["p_gates"], parity_mode=True)
    assert plan.sparse.all()
    phi = O.dense_phi0(g["p_U"])
    v, d, blocks, _ = O.hessian_sum(plan, np.arange(2 ** int(g["p_k"])), phi)
    assert rel_err(plan.logical_sum(d), g["p_holo"]) < 1e-12
    for kk, ref in zip([tuple(x) for x in g["p_hess_keys"]], g["p_hess_blocks"]):
        assert rel_err(blocks[kk], ref) < 1e-12


def test_models_terms_and_lanczos():
    g = golden("models")
    for L, periodic in ((4, False), (4, True), (8, False), (12, False), (14, True), (16, True)):
        key = f"spinful_L{L}_{'p' if periodic else 'o'}"
        terms, groups = O.spinful_terms(L, 1.0, 4.0, periodic)
        arr = np.array([[a, b, c, h] for a, b, c, h in terms], dtype=float)
        assert np.array_equal(arr, g[key + "_terms"])
        assert [len(x) for x in groups] == list(g[key + "_groups"])
    terms, _ = O.spinful_terms(3, 1.0, 4.0, True)
    H = O.HamiltonianApply(6, terms)
    out = O.lanczos_expm(H, g["krylov_in"], 0.25)
    assert rel_err(out, g["krylov_out"]) < 1e-11
    assert rel_err(O.dense_target(6, terms, 0.25) @ g["krylov_in"], g["dense_out"]) < 1e-12


@pytest.mark.slow
def test_c2_slice_lanczos_and_gradient():
    g = golden("c2_slice")
    k = 16
    terms, _ = O.spinful_terms(8, 1.0, 4.0, False)
    phi = O.lanczos_phi0(k, terms, 0.25)
    js = g["js"]
    srng = np.random.default_rng(2)
    srng.choice(2**k, size=16, replace=False)
    w = srng.normal(size=2**k) + 1j * srng.normal(size=2**k)
    P = phi(js[:4])
    for i in range(4):
        chk = [P[i].sum(), P[i] @ w, np.vdot(P[i], P[i]).real]
        assert rel_err(chk, g["phi_checks"][i]) < 1e-10
    plan = O.Plan(k, g["targets"], g["logical"], g["gates"])
    v, d, _ = O.gradient_sum(plan, js[:4], lambda jj: P[np.searchsorted(js[:4], jj)])
    assert abs(v - g["values"][:4].sum()) < 1e-10


def test_reversible_schedule_matches_reference_c1_full_sum():
    """The large-k oracle (reversible 3-vector schedule) against the
    reference's cached-pass drivers: c1 value / gradient / HVP over all 256
    summands."""
    g, U = _c1()
    plan = O.Plan(8, g["targets"], g["logical"], g["gates"])
    phi = O.dense_phi0(U)
    v = 0j
    d = np.zeros((plan.n, 16), complex)
    h = np.zeros((plan.n, 16), complex)
    for j in range(256):
        vj, dj, hj = O.grad_hvp_reversible(plan, list(g["direction"]), j, phi([j])[0])
        v, d, h = v + vj, d + dj, h + hj
    assert abs(-v.real - g["value"]) < 1e-12 * abs(g["value"])
    assert rel_err(plan.logical_sum(d), g["holo"]) < 1e-12
    assert rel_err(plan.logical_sum(h), g["hvp"]) < 1e-12


def test_reversible_schedule_matches_reference_c2_slice():
    """... and on the 16-summand c2 slice the reference drivers produced with
    Krylov targets (phi0 from the Lanczos restatement)."""
    g = golden("c2_slice")
    terms, _ = O.spinful_terms(8, 1.0, 4.0, False)
    js = g["js"]
    P = O.lanczos_phi0(16, terms, 0.25)(js)
    plan = O.Plan(16, g["targets"], g["logical"], g["gates"])
    d = np.zeros((plan.n, 16), complex)
    h = np.zeros((plan.n, 16), complex)
    for i, j in enumerate(js):
        vj, dj, hj = O.grad_hvp_reversible(plan, list(g["direction"]), j, P[i])
        assert abs(vj - g["values"][i]) < 1e-10
        d, h = d + dj, h + hj
    assert rel_err(plan.logical_sum(d), g["holo"]) < 1e-10
    assert rel_err(plan.logical_sum(h), g["hvp"]) < 1e-10
