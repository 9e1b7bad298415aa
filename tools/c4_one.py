"""One BASELINE configs[3] summand (L=14 periodic, sector + fold, k=28):
value + gradient + HVP, for ncu captures of the sector-mode fused passes.
  python tools/c4_one.py [L]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_23775_b200 as gf  # noqa: E402
from oracle import gf_oracle as O  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 14
seed = {14: 3, 16: 4}.get(L, 3)
torch.cuda.set_device(0)
spec, circ, rng = gf.spinful_layer_circuit(L, 9, True, seed=seed, parity=True)
X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), True)
     for g in circ.logical_gates]
k = circ.num_qubits
i0 = int(np.random.default_rng(seed + 1).integers(0, 1 << (k - 1)))
rep_, size = O.orbit_canon(O.sector_unrank(np.array([i0], np.int64), 0), L)
idx = O.sector_rank(rep_)
basis = (idx, size.astype(np.float64))
orc = gf.NumberBlockOracle(spec, 0.25)
cache = gf.models.CachedTargetColumns(orc, k, 0, 1, sector=0, indices=idx, batch=1)
for _ in range(2):
    rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=basis)
torch.cuda.synchronize()
print("c4_one ok", L, rep.value)
