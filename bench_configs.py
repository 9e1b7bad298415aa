#!/usr/bin/env python
"""Per-config measurements for BASELINE.json configs[0], [2], [3], [4] (the
driver's bench.py measures configs[1]).  Each config runs its recipe (SURVEY
Appendix B) on a seeded sample of basis-state summands and reports
summand-evaluations per second with the extrapolated full-sum time; the target
oracle is timed separately.  At full size, a size-independent parity property
is checked: for every slot s, sum_ij G_s[i,j] D_s[i,j] equals the summand sum
phi0 . C|j> (the reinsertion identity, reference test_kernels.py:114-124 /
test_objective.py:115-122).

  python bench_configs.py [c1 c3 c4 c5] > profiles/configs_r01.json
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (L, layers, periodic, parity, sector, fold, seed, sample)
    "c1": (4, 3, False, False, None, False, 0, None),
    "c3": (12, 7, False, True, 0, False, 2, 64),
    "c4": (14, 9, True, True, 0, True, 3, 8),
    "c5": (16, 9, True, True, 0, True, 4, 1),
    "c2h": (8, 5, False, False, None, False, 1, None),   # configs[1]: full Hessian assembly, full 2^16 sum
    "c3tr": (12, 7, False, True, 0, False, 2, 64),       # configs[2]: one TR step, gradient + 10 tCG HVPs
    "c5h": (16, 9, True, True, 0, True, 4, 1),            # configs[4]: one full gradient + 20 HVPs
    "c2hp": (8, 5, False, False, None, False, 1, 1024),   # configs[1] Hessian: pair-CSR vs HVP-column engines
    "bw16d": (8, 5, True, False, None, False, 5, 1024),   # 16-qubit periodic brick wall: translation dedup
}


def run(name):
    import torch

    import paper_2506_23775_b200 as gf
    from paper_2506_23775_b200 import objective as obj

    L, layers, periodic, parity, sector, fold, seed, sample = CONFIGS[name]
    torch.cuda.set_device(0)
    spec, circ, rng = gf.spinful_layer_circuit(L, layers, periodic, seed=seed, parity=parity)
    X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
         for g in circ.logical_gates]
    k = circ.num_qubits
    out = {"config": name, "L": L, "qubits": k, "layers": layers, "slots": circ.num_slots,
           "logical": circ.num_logical, "periodic": periodic, "sector": sector, "fold": fold}
    if name == "c2h":
        orc = gf.ChebyshevOracle(spec, 0.25)
        cache = gf.models.CachedTargetColumns(orc, k, 0, 1 << k, batch=512)
        del orc
        torch.cuda.empty_cache()
        gf.gradient_and_hvp(circ, cache, X)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = gf.full_hessian(circ, cache)
        torch.cuda.synchronize()
        out["full_hessian_s"] = time.perf_counter() - t0
        out["hvp_evaluations"] = circ.num_logical * 16
        out["blocks"] = len(rep.hessian.blocks)
        # size-independent parity: assembled blocks applied to X == engine HVP along X
        hv = gf.hessian_vector_product(circ, cache, X)
        via = rep.hessian.apply_direction(X)
        sc = max(np.abs(np.stack(hv)).max(), 1e-300)
        out["blocks_vs_hvp_max_rel_dev"] = float(max(np.abs(a - b).max() for a, b in zip(via, hv)) / sc)
        diag = [rep.hessian.blocks[(a, a)] for a in range(circ.num_logical) if (a, a) in rep.hessian.blocks]
        out["diag_block_symmetry_max_rel_dev"] = float(max(np.abs(b - b.T).max() / np.abs(b).max() for b in diag))
        out["reference_cpu_estimate_h"] = 149.0  # 8.2 s per summand x 2^16, single core
        return out
    if name in ("c2hp", "bw16d"):
        # full_hessian on a contiguous 1024-summand sample, both engine
        # algorithms (objective.full_hessian method=): the reference's pair-CSR
        # driver (gf_hess_plan_eval) and the HVP-column sweeps; bw16d is a
        # periodic spinless-style brick wall where translation dedup applies
        if name == "bw16d":
            from bench_v1 import IdentityOracle

            grng = np.random.default_rng(seed)
            circ = gf.build_brickwall(16, layers, [gf.manifold.random_unitary(4, grng) for _ in range(layers)],
                                      periodic=True)
            k = 16
            cache = IdentityOracle(k)
            out.update(slots=circ.num_slots, logical=circ.num_logical, qubits=k)
        else:
            cache = gf.models.CachedTargetColumns(gf.NumberBlockOracle(spec, 0.25), k, 0, sample, batch=512)
        basis = (np.arange(sample, dtype=np.int64), None)
        variants = [("columns", False), ("pairs", False)] + ([("pairs", True)] if name == "bw16d" else [])
        ref = None
        for method, dedup in variants:
            kw = dict(method=method, use_translation_dedup=dedup, basis=basis)
            gf.full_hessian(circ, cache, **kw)  # plan + warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = gf.full_hessian(circ, cache, **kw)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            tag = method + ("_dedup" if dedup else "")
            out[f"{tag}_s_per_summand"] = dt / sample
            out[f"{tag}_full_sum_extrapolated_s"] = dt / sample * 2**k
            out[f"{tag}_pass_counts"] = rep.pass_counts
            if ref is None:
                ref = rep
            elif dedup:
                # translation dedup equals the full enumeration only for the full,
                # translation-invariant basis sum -- not for this contiguous sample
                # (checked at full sum against the reference's dedup fixture in
                # tests/test_gpu_api.py); report the work reduction only
                out[f"{tag}_pair_contraction_ratio"] = (rep.pass_counts["pair_contractions"] /
                                                        ref.pass_counts["pair_contractions"])
            else:
                sc = max(np.abs(b).max() for b in ref.hessian.blocks.values())
                out[f"{tag}_vs_columns_max_rel_dev"] = float(max(
                    np.abs(rep.hessian.blocks[kk] - ref.hessian.blocks[kk]).max() for kk in ref.hessian.blocks) / sc)
            obj._PLANS.clear()
            torch.cuda.empty_cache()
        out["sample_summands"] = sample
        return out
    if name == "c1":
        orc = gf.DenseOracle(spec, 0.25)
        for _ in range(3):
            gf.gradient_and_hvp(circ, orc, X)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            rep, hv = gf.gradient_and_hvp(circ, orc, X)
        torch.cuda.synchronize()
        out["full_sum_grad_hvp_s"] = (time.perf_counter() - t0) / reps
        out["value"] = rep.value
        t0 = time.perf_counter()
        final, trace = gf.trust_region_optimize(circ, orc, gf.TrustRegionParams(max_iterations=5))
        out["trust_region_5_iterations_s"] = time.perf_counter() - t0
        out["trust_region_f"] = [r.value for r in trace.records]
        out["reference_cpu_s_survey"] = {"grad": 0.022, "hvp": 0.0317, "tr5": 2.72}
        return out
    sect_size = 1 << (k - 1)
    srng = np.random.default_rng(seed + 1)
    idx = np.unique(srng.integers(0, sect_size, size=sample))
    weights = None
    if fold:
        # canonicalise the sample to orbit representatives with orbit-size weights
        x = torch.from_numpy(idx).cuda()
        full = torch.empty_like(x)
        gf._lib.check(gf._lib.lib.gf_sector_unrank(x.data_ptr(), x.numel(), 0, full.data_ptr(), gf._lib.stream_ptr()))
        rep, size = torch.empty_like(full), torch.empty_like(full)
        gf._lib.check(gf._lib.lib.gf_orbit_canon(full.data_ptr(), full.numel(), L, rep.data_ptr(), size.data_ptr(),
                                                 gf._lib.stream_ptr()))
        comp = torch.empty_like(rep)
        gf._lib.check(gf._lib.lib.gf_sector_rank(rep.data_ptr(), rep.numel(), comp.data_ptr(), gf._lib.stream_ptr()))
        idx, first = np.unique(comp.cpu().numpy(), return_index=True)
        weights = size.cpu().numpy()[first].astype(np.float64)
        out["orbit_reps_total_burnside"] = {14: 19173968, 16: 268443720}.get(L)
    out["sample_summands"] = int(idx.size)
    # target columns of the sample: number-block Chebyshev oracle (each
    # column inside its particle-number block), timed separately
    orc = gf.NumberBlockOracle(spec, 0.25)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = gf.models.CachedTargetColumns(orc, k, 0, idx.size, sector=0, indices=idx, batch=1)
    torch.cuda.synchronize()
    out["oracle_s_per_summand"] = (time.perf_counter() - t0) / idx.size
    out["oracle_chebyshev_order"] = orc.order
    out["oracle"] = type(orc).__name__
    # cross-check one column against the full-space Chebyshev oracle
    chk = gf.ChebyshevOracle(spec, 0.25)
    first = torch.from_numpy(idx[:1]).cuda()
    jf = torch.empty_like(first)
    gf._lib.check(gf._lib.lib.gf_sector_unrank(first.data_ptr(), 1, 0, jf.data_ptr(), gf._lib.stream_ptr()))
    col = torch.empty((1, sect_size), dtype=torch.complex128, device="cuda")
    chk.phi0_into(jf, 0, col)
    out["oracle_vs_full_space_chebyshev_max_abs"] = float(torch.max(torch.abs(col - cache.rows[:1])).item())
    del chk, col
    del orc
    torch.cuda.empty_cache()
    basis = (idx, weights)
    rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)  # warm-up + plan
    plan = list(obj._PLANS.values())[-1]
    out["engine"] = plan.describe()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 2 if k >= 28 else 3
    for _ in range(reps):
        rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out["grad_hvp_s_per_summand"] = dt / idx.size
    out["summand_evals_per_s"] = idx.size / dt
    total = out.get("orbit_reps_total_burnside") or sect_size
    out["full_sum_summands"] = total
    out["extrapolated_full_sum_grad_hvp_hours_1gpu"] = total * dt / idx.size / 3600
    if name == "c5h":
        # configs[4] as stated: one gradient + 20 HVPs per summand, the HVPs in
        # multi-direction sweeps (as many directions per sweep as fit in HBM)
        dirs = []
        for _ in range(20):
            dirs.append([gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) +
                                                          1j * rng.normal(size=(4, 4)), True)
                         for g in circ.logical_gates])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gf.full_gradient(circ, cache, parity_mode=True, sector=0, basis=basis)
        torch.cuda.synchronize()
        out["gradient_s_per_summand"] = (time.perf_counter() - t0) / idx.size
        t0 = time.perf_counter()
        hv20 = gf.hessian_vector_products(circ, cache, dirs, sector=0, basis=basis)
        torch.cuda.synchronize()
        out["hvp20_s_per_summand"] = (time.perf_counter() - t0) / idx.size
        out["directions_per_sweep"] = obj._directions_per_sweep(circ, 0)
        out["gradient_plus_20_hvp_s_per_summand"] = out["gradient_s_per_summand"] + out["hvp20_s_per_summand"]
        # consistency: direction 0 of the batched sweeps equals the single-direction HVP
        single = gf.hessian_vector_product(circ, cache, dirs[0], sector=0, basis=basis)
        sc = max(np.abs(np.stack(single)).max(), 1e-300)
        out["multi_vs_single_hvp_max_rel_dev"] = float(np.abs(np.stack(hv20[0]) - np.stack(single)).max() / sc)
        return out
    if name == "c3tr":
        # configs[2] as stated: gradient + 10 HVPs per TR step, timed directly
        # (the tCG of a real step may stop earlier at the boundary / negative
        # curvature; the TR step below reports its own inner count)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gf.full_gradient(circ, cache, parity_mode=True, sector=0, basis=basis)
        for _ in range(10):
            gf.hessian_vector_product(circ, cache, X, sector=0, basis=basis)
        torch.cuda.synchronize()
        out["gradient_plus_10_hvp_s"] = time.perf_counter() - t0
        out["gradient_plus_10_hvp_s_per_summand"] = out["gradient_plus_10_hvp_s"] / idx.size
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        params = gf.TrustRegionParams(max_iterations=1, use_hvp=True, tcg=gf.TcgParams(max_inner=10))
        final, trace = gf.trust_region_optimize(circ, cache, params, parity_mode=True, sector=0, basis=basis)
        torch.cuda.synchronize()
        r = trace.records[0]
        out["tr_step_s"] = time.perf_counter() - t0
        out["tr_inner_iterations"] = r.inner_iterations
        out["tr_stop_reason"] = r.stop_reason
        out["tr_engine_evaluations"] = 1 + r.inner_iterations + 1 + 1  # gradient, tCG HVPs, model HVP, value
        return out
    # HVP-only (tCG inner step) throughput
    t0 = time.perf_counter()
    hv2 = gf.hessian_vector_product(circ, cache, X, sector=0, basis=basis)
    torch.cuda.synchronize()
    out["hvp_s_per_summand"] = (time.perf_counter() - t0) / idx.size
    # size-independent parity: reinsertion identity per slot on the last batch
    nlast = idx.size - ((idx.size - 1) // plan.batch) * plan.batch
    gf.full_gradient(circ, cache, parity_mode=True, sector=0, basis=(idx[-nlast:], None if weights is None
                                                                       else weights[-nlast:]))
    d, _ = plan.slot_outputs(nlast)
    run_v = gf.target_value(circ, cache, sector=0, basis=(idx[-nlast:], None if weights is None
                                                          else weights[-nlast:]))
    vals = []
    t1, t2, lid = circ.slot_arrays()
    for s in range(circ.num_slots):
        gm = circ.logical_gates[lid[s]].matrix
        if t1[s] > t2[s]:
            gm = gf.kernels.wire_swapped_matrix(gm)
        vals.append(np.sum(gm * d[s]))
    vals = np.array(vals)
    out["reinsertion_max_rel_dev"] = float(np.max(np.abs(-vals.real - run_v)) / max(1.0, abs(run_v)))
    out["value_sample"] = rep.value
    return out


if __name__ == "__main__":
    import subprocess

    if len(sys.argv) == 3 and sys.argv[1] == "--one":
        print(json.dumps(run(sys.argv[2])), flush=True)
        sys.exit(0)
    names = sys.argv[1:] or ["c1", "c3", "c4", "c5", "c2h", "c3tr"]
    for nm in names:  # one process per config: each frees its device memory on exit
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", nm], capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps(
            {"config": nm, "error": r.stderr.strip().splitlines()[-1] if r.stderr.strip() else "no output"})
        print(line, flush=True)
