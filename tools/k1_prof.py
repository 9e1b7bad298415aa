"""Run a few K1 gate applications on a 2^31 vector (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_23775_b200 as gf

K = 31
x = torch.empty(1 << K, dtype=torch.complex128, device="cuda")
x.real.normal_()
x.imag.normal_()
st = gf._lib.stream_ptr()
rng = np.random.default_rng(0)
for a, b in ((29, 30), (28, 29), (10, 11), (15, 30), (3, 18)):
    g = np.ascontiguousarray(gf.manifold.random_unitary(4, rng))
    gf._lib.check(gf._lib.lib.gf_apply_gate(x.data_ptr(), x.data_ptr(), K, a, b, g.ctypes.data, 0, 1, st))
g = np.ascontiguousarray(gf.manifold.parity_join(gf.manifold.random_unitary(2, rng), gf.manifold.random_unitary(2, rng)))
gf._lib.check(gf._lib.lib.gf_apply_gate_sector_c1q(x.data_ptr(), x.data_ptr(), K + 1, 20, 0, g.ctypes.data, 1, st))
torch.cuda.synchronize()
