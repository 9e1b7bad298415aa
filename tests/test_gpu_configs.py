"""BASELINE configs at their stated sizes against independent paths (GPU).

* c2 (configs[1]): 1024 seeded summands on the bench's plan (the exact 3-pass
  plan; batch 512, two batches -- the bench runs batches of 2048) against the CPU oracle port of the
  reference's cached-pass drivers (_gradient_chunk / _hvp_chunk,
  objective.py:322-337, 432-482).
* c3 (configs[2]): L=12 open, 24 qubits, even sector compressed to 2^23
  amplitudes, 80 slots.  Two seeded sector summands through the engine
  (parity-controlled 1q slots, fused passes at high global bits) against the
  oracle's reversible schedule in the FULL 2^24 space -- the reference
  semantics restricted to the sector's basis states.
* c4 / c5 (configs[3], [4]): one folded orbit representative each (k = 28 /
  32, 2^27 / 2^31 compressed amplitudes) through the fused tile engine and
  through the independent streaming engine (GF_ENGINE=stream: one launch per
  slot, FMA gate and hole kernels) on the same inputs.

Tolerance: the north-star 1e-10 relative (max-abs over entries).  Target
columns come from the GPU Chebyshev / number-block oracles (pinned against the
reference Krylov and dense oracles in test_gpu_engine.py); both sides of each
comparison get the same columns.
"""

import numpy as np
import pytest

from conftest import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2506_23775_b200 as gf  # noqa: E402
from paper_2506_23775_b200 import objective as obj  # noqa: E402
from oracle import gf_oracle as O  # noqa: E402

TOL = 1e-10


def _recipe(L, layers, periodic, seed, parity):
    spec, circ, rng = gf.spinful_layer_circuit(L, layers, periodic, seed=seed, parity=parity)
    X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), parity)
         for g in circ.logical_gates]
    return spec, circ, X


def _oracle_plan(circ):
    t1, t2, lid = circ.slot_arrays()
    return O.Plan(circ.num_qubits, np.stack([t1, t2], 1), lid, circ.gate_stack())


def _free_gib():
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


def test_c2_1024_summands_bench_shape_vs_oracle_port():
    spec, circ, X = _recipe(8, 5, False, 1, False)
    k = 16
    idx = np.sort(np.random.default_rng(21).choice(1 << k, size=1024, replace=False)).astype(np.int64)
    orc = gf.NumberBlockOracle(spec, 0.25)
    cache = gf.models.CachedTargetColumns(orc, k, 0, idx.size, indices=idx, batch=512)
    rep, hv = gf.gradient_and_hvp(circ, cache, X, basis=(idx, None), batch=512)
    plan = list(obj._PLANS.values())[-1]
    assert plan.batch == 512 and plan.describe()["rev_passes"] in (3, 4)  # the bench's plan (it runs batches of 2048)
    P = cache.rows.cpu().numpy()
    oplan = _oracle_plan(circ)
    fn = lambda jj: P[np.searchsorted(idx, jj)]
    v, d, _ = O.gradient_sum(oplan, idx, fn, workers=16)
    h, _ = O.hvp_sum(oplan, X, idx, fn, workers=16)
    assert abs(rep.value + v.real) <= TOL * max(1.0, abs(v.real))
    assert rel_err(np.stack(rep.holomorphic_derivatives), oplan.logical_sum(d)) < TOL
    assert rel_err(np.stack(hv), oplan.logical_sum(h)) < TOL


def test_c3_sector_summands_vs_full_space_reversible_oracle():
    spec, circ, X = _recipe(12, 7, False, 2, True)
    k = 24
    assert circ.num_slots == 80
    idx = np.sort(np.random.default_rng(3).choice(1 << (k - 1), size=2, replace=False)).astype(np.int64)
    js = O.sector_unrank(idx, 0)
    orc = gf.ChebyshevOracle(spec, 0.25)
    full = torch.empty((2, 1 << k), dtype=torch.complex128, device="cuda")
    orc.phi0_into(torch.from_numpy(js).cuda(), None, full)
    # the engine gets the sector rows of the same columns
    comp = full[:, _sector_sel(k)]
    cache = _RowsOracle(orc, comp.contiguous(), idx)
    rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=(idx, None))
    F = full.cpu().numpy()
    del full, comp, cache
    obj._PLANS.clear()
    torch.cuda.empty_cache()
    oplan = _oracle_plan(circ)
    v = 0j
    d = np.zeros((oplan.n, 16), complex)
    h = np.zeros((oplan.n, 16), complex)
    for i, j in enumerate(js):
        vj, dj, hj = O.grad_hvp_reversible(oplan, X, int(j), F[i])
        v, d, h = v + vj, d + dj, h + hj
    assert abs(rep.value + v.real) <= TOL * abs(v)
    assert rel_err(np.stack(rep.holomorphic_derivatives), oplan.logical_sum(d)) < TOL
    assert rel_err(np.stack(hv), oplan.logical_sum(h)) < TOL


def _sector_sel(k):
    sel = O.sector_unrank(np.arange(1 << (k - 1), dtype=np.int64), 0)
    return torch.from_numpy(sel).cuda()


class _RowsOracle:
    """Duck-typed oracle handing the engine precomputed sector rows."""

    def __init__(self, inner, rows, idx):
        self.num_qubits = inner.num_qubits
        self.inner = inner
        self.rows = rows
        self.idx = idx

    def apply(self, s):
        return self.inner.apply(s)

    def apply_adjoint(self, s):
        return self.inner.apply_adjoint(s)

    def phi0_at(self, pos, nvec, sector_code, indices=None):
        if sector_code != 0 or indices is None or not np.array_equal(indices[pos:pos + nvec], self.idx[pos:pos + nvec]):
            return None
        return self.rows[pos:pos + nvec]


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_folded_summand_fused_vs_streaming_engine(monkeypatch, name):
    L, seed, need = {"c4": (14, 3, 20), "c5": (16, 4, 140)}[name]
    if _free_gib() < need:
        pytest.skip(f"needs {need} GiB free device memory")
    spec, circ, X = _recipe(L, 9, True, seed, True)
    k = circ.num_qubits
    i0 = int(np.random.default_rng(seed + 1).integers(0, 1 << (k - 1)))
    full = O.sector_unrank(np.array([i0], np.int64), 0)
    rep_, size = O.orbit_canon(full, L)
    idx = O.sector_rank(rep_)
    basis = (idx, size.astype(np.float64))
    orc = gf.NumberBlockOracle(spec, 0.25)
    cache = gf.models.CachedTargetColumns(orc, k, 0, 1, sector=0, indices=idx, batch=1)
    del orc
    torch.cuda.empty_cache()
    res = {}
    for eng in ("fused", "stream"):
        if eng == "stream":
            monkeypatch.setenv("GF_ENGINE", "stream")
        obj._PLANS.clear()
        torch.cuda.empty_cache()
        rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)
        res[eng] = (rep.value, np.stack(rep.holomorphic_derivatives), np.stack(hv))
        assert list(obj._PLANS.values())[-1].describe()["fused"] == (eng == "fused")
    obj._PLANS.clear()
    del cache
    torch.cuda.empty_cache()
    (vf, df, hf), (vs, ds, hs) = res["fused"], res["stream"]
    assert abs(vf - vs) <= TOL * abs(vs)
    assert rel_err(df, ds) < TOL
    assert rel_err(hf, hs) < TOL
