import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2506_23775_b200 as gf
spec, circ, rng = gf.spinful_layer_circuit(16, 9, True, seed=4, parity=True)
X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), True) for g in circ.logical_gates]
orc = gf.ChebyshevOracle(spec, 0.25)
idx = np.array([12345], dtype=np.int64)
cache = gf.models.CachedTargetColumns(orc, 32, 0, 1, sector=0, indices=idx, batch=1)
del orc; torch.cuda.empty_cache()
rep, hv = gf.gradient_and_hvp(circ, cache, X, parity_mode=True, sector=0, basis=(idx, None))
torch.cuda.synchronize()
print("ok", rep.value)
