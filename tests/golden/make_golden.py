"""Generate golden fixtures by running the UNMODIFIED reference (`gatefit`).

Test infrastructure only: this script imports the reference package from
``/root/reference/pkg/src`` (read-only; numba's cache is redirected to /tmp so
nothing is written into the reference tree) and stores its outputs as small
``.npz`` fixtures next to this file.  The fixtures pin the CPU oracle in
``oracle/`` and the CUDA engine; nothing at test/bench time on the GPU box reads
``/root/reference``.

Config recipes follow SURVEY.md Appendix B.1 (spinful Fermi-Hubbard groups from
``models.build_spinful_fh`` -- reference models.py:149-170 -- one logical gate
per layer, layer i uses group i mod 3) and BASELINE.json configs[0..1].

Run:  python tests/golden/make_golden.py   (takes ~2-3 minutes)
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gf_numba_cache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from gatefit import circuit as C  # noqa: E402
from gatefit import kernels as K  # noqa: E402
from gatefit import manifold, models, objective, optimizer  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def spinful_layers(L, nlayers, periodic, rng, parity=False):
    """SURVEY Appendix B.1 recipe: layer i -> Trotter group i mod 3."""
    spec = models.build_spinful_fh(L, 1.0, 4.0, periodic)
    groups = spec.trotter_groups
    slots, gates = [], []
    for layer in range(nlayers):
        g = groups[layer % len(groups)]
        if parity:
            m = manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng))
        else:
            m = manifold.random_unitary(4, rng)
        gates.append(K.Gate(m, g.bonds[0], parity_sparse=parity))
        for b in g.bonds:
            slots.append(C.GateSlot(layer, b))
    return spec, C.Circuit(spec.num_qubits, slots, gates)


def circ_arrays(circ):
    return dict(
        k=circ.num_qubits,
        targets=np.array([s.targets for s in circ.slots], dtype=np.int64).reshape(-1, 2),
        logical=np.array([s.logical_id for s in circ.slots], dtype=np.int64),
        gates=np.stack([g.matrix for g in circ.logical_gates]),
    )


def tangent_dirs(circ, rng, parity=False):
    return [
        manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
        for g in circ.logical_gates
    ]


def hessian_dict(rep, prefix):
    out = {}
    keys = sorted(rep.hessian.blocks)
    out[prefix + "keys"] = np.array(keys, dtype=np.int64).reshape(-1, 2)
    out[prefix + "blocks"] = np.stack([rep.hessian.blocks[k] for k in keys]) if keys else np.zeros((0, 16, 16))
    out[prefix + "support"] = np.asarray(rep.hessian.support)
    return out


# ---------------------------------------------------------------------------


def gen_kernels():
    """Kernel-level vectors (reference kernels.py:484-623)."""
    rng = np.random.default_rng(11)
    k = 5
    N = 2**k
    pairs = [(0, 1), (1, 0), (0, 4), (4, 0), (2, 3), (3, 1), (1, 4), (4, 3), (0, 2)]
    psi = rng.normal(size=N) + 1j * rng.normal(size=N)
    bra = rng.normal(size=N) + 1j * rng.normal(size=N)
    out = dict(k=k, pairs=np.array(pairs), psi=psi, bra=bra)
    gm, pm = [], []
    ap, app, hc, ha, hap, aa, hca, hcap = [], [], [], [], [], [], [], []
    for t in pairs:
        g = manifold.random_unitary(4, rng)
        p = manifold.parity_join(manifold.random_unitary(2, rng), manifold.random_unitary(2, rng))
        gm.append(g)
        pm.append(p)
        ap.append(K.apply_gate(psi, K.Gate(g, t)))
        app.append(K.apply_gate(psi, K.Gate(p, t)))
        hc.append(K.hole_contract(bra, psi, t))
        arr = K.hole_apply(psi, t)
        ha.append(arr)
        arrp = K.hole_apply(psi, t, support=K.PARITY_SUPPORT)
        hap.append(arrp)
        t2 = pairs[(pairs.index(t) + 3) % len(pairs)]
        aa.append(K.apply_gate_to_array(arr, K.Gate(g, t2)))
        hca.append(K.hole_contract_array(bra, arr, t2))
        hcap.append(K.hole_contract_array(bra, arrp, t2, support=K.PARITY_SUPPORT))
    out.update(
        gates=np.stack(gm), pgates=np.stack(pm), apply=np.stack(ap), apply_parity=np.stack(app),
        hole_contract=np.stack(hc), hole_apply=np.stack(ha), hole_apply_parity=np.stack(hap),
        array_apply=np.stack(aa), hole_contract_array=np.stack(hca),
        hole_contract_array_parity=np.stack(hcap),
        second_pairs=np.array([pairs[(i + 3) % len(pairs)] for i in range(len(pairs))]),
    )
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def gen_c1():
    """BASELINE configs[0]: L=4 open spinful FH, 3 layers, Haar seed 0, t=0.25."""
    rng = np.random.default_rng(0)
    spec, circ = spinful_layers(4, 3, False, rng)
    orc = models.make_oracle(spec, 0.25, "dense")
    X = tangent_dirs(circ, rng)
    grad = objective.full_gradient(circ, orc)
    hvp = objective.hessian_vector_product(circ, orc, X)
    hess = objective.full_hessian(circ, orc)
    hx = [
        manifold.hessian_apply_gate(g.matrix, e, manifold.euclid_gradient_from_holomorphic(h), x)
        for g, e, h, x in zip(circ.logical_gates, grad.euclidean_gradients, hvp, X)
    ]
    tv = objective.target_value(circ, orc)
    params = optimizer.TrustRegionParams(max_iterations=5)
    t0 = time.time()
    final, trace = optimizer.trust_region_optimize(circ, orc, params)
    tr_s = time.time() - t0
    rec = trace.records
    out = circ_arrays(circ)
    out.update(
        U_cols=orc._u[:, :4].copy(),
        U_diag=np.diag(orc._u).copy(),
        value=grad.value,
        target_value=tv,
        holo=np.stack(grad.holomorphic_derivatives),
        euclid=np.stack(grad.euclidean_gradients),
        riem=np.stack(grad.per_logical_gradient),
        direction=np.stack(X),
        hvp=np.stack(hvp),
        hess_x=np.stack(hx),
        x_hess_x=sum(manifold.inner(x, y) for x, y in zip(X, hx)),
        grad_counts=np.array([grad.pass_counts[n] for n in objective._COUNT_NAMES]),
        hess_counts=np.array([hess.pass_counts[n] for n in objective._COUNT_NAMES]),
        hess_value=hess.value,
        tr_f=np.array([r.value for r in rec]),
        tr_rho=np.array([r.rho for r in rec]),
        tr_radius=np.array([r.radius for r in rec]),
        tr_gnorm=np.array([r.grad_norm for r in rec]),
        tr_step=np.array([r.step_norm for r in rec]),
        tr_inner=np.array([r.inner_iterations for r in rec]),
        tr_accepted=np.array([r.accepted for r in rec]),
        tr_reason=np.array([r.stop_reason for r in rec]),
        tr_final_gates=np.stack([g.matrix for g in final.logical_gates]),
        tr_seconds_ref=tr_s,
    )
    out.update(hessian_dict(hess, "hess_"))
    np.savez_compressed(os.path.join(HERE, "c1.npz"), **out)
    print("c1 value", grad.value, "TR", out["tr_f"])


def gen_c2_slice():
    """BASELINE configs[1] (L=8, 16 qubits, 5 layers, Haar seed 1) on a seeded
    sample of 16 basis states: the reference chunk drivers
    (objective.py:322-337 gradient, objective.py:432-482 hvp) with phi0 from the
    reference KrylovOracle (models.py:322-384; the dense one refuses k=16)."""
    rng = np.random.default_rng(1)
    spec, circ = spinful_layers(8, 5, False, rng)
    X = tangent_dirs(circ, rng)
    k = circ.num_qubits
    N = 2**k
    srng = np.random.default_rng(2)
    js = np.sort(srng.choice(N, size=16, replace=False))
    orc = models.make_oracle(spec, 0.25, "krylov")
    w = srng.normal(size=N) + 1j * srng.normal(size=N)
    plan = objective._Plan(circ, False)
    n = circ.num_slots
    zm = np.empty((n, 4, 4), complex)
    for i, s in enumerate(circ.slots):
        z = X[s.logical_id]
        if plan.swapped[i]:
            z = K.wire_swapped_matrix(z)
        zm[i] = z
    zmt = np.ascontiguousarray(np.transpose(zm, (0, 2, 1)))
    vals, dsum, hsum, phichk = [], np.zeros((n, 4, 4), complex), np.zeros((n, 4, 4), complex), []
    for j in js:
        phi0 = np.conj(orc.apply(K.basis_state(k, int(j))))[None, :]
        phichk.append([phi0[0].sum(), phi0[0] @ w, np.vdot(phi0[0], phi0[0]).real])
        counts = np.zeros(5, np.int64)
        psis = np.empty((n + 1, N), complex)
        phis = np.empty((n + 1, N), complex)
        dacc = np.zeros((n, 4, 4), complex)
        v = objective._gradient_chunk(plan.mats, plan.mats_t, plan.adjacent, plan.sparse, plan.ps, plan.qs,
                                      plan.ns, int(j), int(j) + 1, phi0, psis, phis, dacc, counts)
        oacc = np.zeros((n, 4, 4), complex)
        objective._hvp_chunk(plan.mats, plan.mats_t, plan.adjacent, plan.sparse, plan.ps, plan.qs, plan.ns,
                             zm, zmt, int(j), int(j) + 1, phi0, psis, phis, np.empty(N, complex),
                             np.empty(N, complex), oacc, counts)
        vals.append(v)
        dsum += dacc
        hsum += oacc
    holo = objective._logical_derivatives(plan, circ, dsum)
    hvp = objective._logical_derivatives(plan, circ, hsum)
    out = circ_arrays(circ)
    # the checksum weight vector w is regenerated from default_rng(2) by the tests
    out.update(js=js, values=np.array(vals), holo=np.stack(holo), hvp=np.stack(hvp),
               direction=np.stack(X), phi_checks=np.array(phichk))
    np.savez_compressed(os.path.join(HERE, "c2_slice.npz"), **out)
    print("c2 slice value sum", np.sum(vals))


def _per_j_sums(circ, orc, js, X, parity_mode):
    """Sum of the reference per-summand drivers over an explicit index set.
    This is the derived oracle for sector-restricted sums."""
    k = circ.num_qubits
    N = 2**k
    n = circ.num_slots
    plan = objective._Plan(circ, parity_mode)
    zplan = objective._Plan(circ, False)
    zm = np.empty((n, 4, 4), complex)
    for i, s in enumerate(circ.slots):
        z = X[s.logical_id]
        if zplan.swapped[i]:
            z = K.wire_swapped_matrix(z)
        zm[i] = z
    zmt = np.ascontiguousarray(np.transpose(zm, (0, 2, 1)))
    val = 0j
    dsum = np.zeros((n, 4, 4), complex)
    hsum = np.zeros((n, 4, 4), complex)
    psis = np.empty((n + 1, N), complex)
    phis = np.empty((n + 1, N), complex)
    counts = np.zeros(5, np.int64)
    for j in js:
        phi0 = np.conj(orc.apply(K.basis_state(k, int(j))))[None, :]
        val += objective._gradient_chunk(plan.mats, plan.mats_t, plan.adjacent, plan.sparse, plan.ps,
                                         plan.qs, plan.ns, int(j), int(j) + 1, phi0, psis, phis, dsum, counts)
        objective._hvp_chunk(zplan.mats, zplan.mats_t, zplan.adjacent, zplan.sparse, zplan.ps, zplan.qs,
                             zplan.ns, zm, zmt, int(j), int(j) + 1, phi0, psis, phis, np.empty(N, complex),
                             np.empty(N, complex), hsum, counts)
    holo = objective._logical_derivatives(plan, circ, dsum)
    hvp = objective._logical_derivatives(zplan, circ, hsum)
    return val, np.stack(holo), np.stack(hvp)


def gen_sector(L, nlayers, periodic, seed, name):
    """Parity-sector restricted sums (no reference implementation: derived
    from the reference drivers run over the even / odd index sets)."""
    rng = np.random.default_rng(seed)
    spec, circ = spinful_layers(L, nlayers, periodic, rng, parity=True)
    X = tangent_dirs(circ, rng, parity=True)
    orc = models.make_oracle(spec, 0.25, "dense")
    k = circ.num_qubits
    N = 2**k
    par = np.array([bin(j).count("1") & 1 for j in range(N)])
    out = circ_arrays(circ)
    out["direction"] = np.stack(X)
    for sect, name_s in ((0, "even"), (1, "odd")):
        js = np.nonzero(par == sect)[0]
        v, h, z = _per_j_sums(circ, orc, js, X, True)
        out[name_s + "_value"] = v
        out[name_s + "_holo"] = h
        out[name_s + "_hvp"] = z
    full = objective.full_gradient(circ, orc, parity_mode=True)
    out["full_value"] = full.value
    out["full_holo"] = np.stack(full.holomorphic_derivatives)
    out["full_hvp"] = np.stack(objective.hessian_vector_product(circ, orc, X))
    out["periodic"] = periodic
    out["L"] = L
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "even value", out["even_value"])


def gen_dedup():
    """Spinless periodic brick wall (k=6) full Hessian with and without the
    reference's translation-class dedup (objective.py:209-247), parity mode
    on a Trotter circuit, and worker-count determinism inputs."""
    rng = np.random.default_rng(7)
    gates = [manifold.random_unitary(4, rng) for _ in range(3)]
    circ = C.build_brickwall(6, 3, gates, periodic=True)
    orc = models.make_oracle(models.build_spinless_fh(6, 1.0, 4.0, periodic=True), 0.4, "dense")
    full = objective.full_hessian(circ, orc, use_translation_dedup=False)
    dd = objective.full_hessian(circ, orc, use_translation_dedup=True)
    classes = C.translation_classes(circ)
    out = circ_arrays(circ)
    out.update(U=orc._u, value=full.value, holo=np.stack(full.holomorphic_derivatives))
    out.update(hessian_dict(full, "full_"))
    out.update(hessian_dict(dd, "dedup_"))
    out["classes"] = np.array([[a, b, m] for (a, b), m in classes], dtype=np.int64)
    out["full_counts"] = np.array([full.pass_counts[n] for n in objective._COUNT_NAMES])
    out["dedup_counts"] = np.array([dd.pass_counts[n] for n in objective._COUNT_NAMES])
    # parity-mode Hessian of a Trotter circuit (parity-sparse kernels, A=8)
    spec = models.build_spinless_fh(4, 1.0, 4.0, periodic=True)
    porc = models.make_oracle(spec, 0.3, "dense")
    pc = models.build_trotter_circuit(spec, models.TrotterPlan(2, 1, 0.3))
    prep = objective.full_hessian(pc, porc, parity_mode=True)
    out.update({"p_" + k: v for k, v in circ_arrays(pc).items()})
    out["p_U"] = porc._u
    out["p_value"] = prep.value
    out["p_holo"] = np.stack(prep.holomorphic_derivatives)
    out["p_riem"] = np.stack(prep.per_logical_gradient)
    out.update(hessian_dict(prep, "p_hess_"))
    np.savez_compressed(os.path.join(HERE, "dedup.npz"), **out)
    print("dedup classes", len(classes))


def gen_models():
    """Model/Trotter/oracle anchors (reference models.py)."""
    out = {}
    for L, periodic in ((4, False), (4, True), (8, False), (12, False), (14, True), (16, True)):
        spec = models.build_spinful_fh(L, 1.0, 4.0, periodic)
        key = f"spinful_L{L}_{'p' if periodic else 'o'}"
        out[key + "_terms"] = np.array([[t.sites[0], t.sites[1], t.coefficient, t.operator == "hop"]
                                        for t in spec.terms], dtype=float)
        out[key + "_groups"] = np.array([len(g.bonds) for g in spec.trotter_groups])
    spec = models.build_spinful_fh(2, 1.0, 4.0, False)
    out["spinful_L2_H"] = models.dense_hamiltonian(spec)
    spec = models.build_spinless_fh(6, 1.0, 4.0, True)
    plan = models.TrotterPlan(4, 1, 0.3)
    circ = models.build_trotter_circuit(spec, plan)
    out["trotter4_spinless6_ngates"] = circ.num_logical
    out["trotter4_spinless6_gates"] = np.stack([g.matrix for g in circ.logical_gates])
    out["trotter4_spinless6_targets"] = np.array([s.targets for s in circ.slots])
    out["trotter4_spinless6_logical"] = np.array([s.logical_id for s in circ.slots])
    rng = np.random.default_rng(3)
    spec = models.build_spinful_fh(3, 1.0, 4.0, True)
    st = rng.normal(size=64) + 1j * rng.normal(size=64)
    out["krylov_in"] = st
    out["krylov_out"] = models.KrylovOracle(spec, 0.25).apply(st)
    out["dense_out"] = models.DenseOracle(spec, 0.25).apply(st)
    np.savez_compressed(os.path.join(HERE, "models.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "c1", "sector", "dedup", "models", "c2"]
    t0 = time.time()
    if "kernels" in which:
        gen_kernels()
    if "c1" in which:
        gen_c1()
    if "sector" in which:
        gen_sector(4, 3, True, 2, "sector_l4p")
        gen_sector(6, 3, True, 4, "sector_l6p")
        gen_sector(5, 4, False, 5, "sector_l5o")
    if "dedup" in which:
        gen_dedup()
    if "models" in which:
        gen_models()
    if "c2" in which:
        gen_c2_slice()
    print("done in %.1fs" % (time.time() - t0))
