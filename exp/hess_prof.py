import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2506_23775_b200 as gf
spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
orc = gf.ChebyshevOracle(spec, 0.25)
cache = gf.models.CachedTargetColumns(orc, 16, 0, 1024, batch=512)
nlog = circ.num_logical
dirs = []
for e in range(3):
    z = np.zeros((nlog, 4, 4), complex); z[2].reshape(16)[e] = 1.0; dirs.append(z)
basis = np.arange(1024)
for _ in range(2):
    gf.hessian_vector_products(circ, cache, dirs, basis=basis)
    gf.hessian_vector_product(circ, cache, dirs[0], basis=basis)
torch.cuda.synchronize()
import time
t0 = time.perf_counter(); gf.hessian_vector_products(circ, cache, dirs, basis=basis); torch.cuda.synchronize(); t1 = time.perf_counter()
gf.hessian_vector_product(circ, cache, dirs[0], basis=basis); torch.cuda.synchronize(); t2 = time.perf_counter()
print("multi3 %.3f s   single %.3f s" % (t1 - t0, t2 - t1))
