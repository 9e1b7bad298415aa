import time, torch, numpy as np
import paper_2506_23775_b200 as gf
from paper_2506_23775_b200 import _lib
spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
o = gf.NumberBlockOracle(spec, 0.25)
o._tables()
torch.cuda.synchronize()
# host part: monkeypatch the launches out
real = _lib.lib.gf_nb_block_matrix
class Fake:
    def __getattr__(self, n): return getattr(_lib.lib_real, n)
for rep in range(2):
    o2 = gf.NumberBlockOracle(spec, 0.25)
    t = time.perf_counter(); o2._tables(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"_tables host-return {t1-t:.3f}s, +sync {t2-t1:.3f}s")
# GPU time per block via events
keys = [(a, b) for a in range(9) for b in range(9)]
coefs = torch.from_numpy(np.ascontiguousarray(o.coef, np.complex128)).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for (a, b) in [(4, 4), (3, 4), (2, 2)]:
    D = o.block_dim((a, b)); out = torch.empty((D, D), dtype=torch.complex128, device="cuda"); desc = o._desc((a, b))
    for r in range(2):
        e0.record()
        _lib.check(_lib.lib.gf_nb_block_matrix(out.data_ptr(), desc.ctypes.data, len(desc), o._nb_terms.ctypes.data,
                                               o._nb_coef.ctypes.data, len(o._nb_coef), coefs.data_ptr(), o.order,
                                               1.0 / o.b, -o.a / o.b, _lib.stream_ptr()))
        e1.record(); torch.cuda.synchronize()
    print("block", (a, b), "D", D, "ms", e0.elapsed_time(e1))
