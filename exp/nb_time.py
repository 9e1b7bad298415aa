import time, torch, numpy as np
import paper_2506_23775_b200 as gf
spec, circ, rng = gf.spinful_layer_circuit(8, 5, False, seed=1)
for rep in range(2):
    torch.cuda.synchronize(); t=time.perf_counter()
    o = gf.NumberBlockOracle(spec, 0.25)
    o._tables(); torch.cuda.synchronize(); t1=time.perf_counter()
    out = torch.empty((512, 65536), dtype=torch.complex128, device="cuda")
    for s in range(0, 65536, 512):
        o.phi0_into(torch.arange(s, s+512, device="cuda"), None, out)
    torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"tables {t1-t:.3f}s  128 batch fills {t2-t1:.3f}s")
c = gf.ChebyshevOracle(spec, 0.25)
ref = torch.empty_like(out)
js = torch.arange(65536-512, 65536, device="cuda")
c.phi0_into(js, None, ref)
print("max diff vs full-space Chebyshev", torch.max(torch.abs(ref-out)).item())
