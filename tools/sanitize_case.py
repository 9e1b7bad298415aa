"""Small engine workload for compute-sanitizer (memcheck / racecheck /
synccheck): k=12 spinful circuit with forced 2^7 tiles (multi-tile,
multi-pass fused plans), value + gradient + HVP, a 3-direction HVP sweep, a
sector-compressed evaluation, and the kernel-level ops.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GF_FUSED_M", "7")

import torch  # noqa: E402

import paper_2506_23775_b200 as gf  # noqa: E402

torch.cuda.set_device(0)
spec, circ, rng = gf.spinful_layer_circuit(6, 4, False, seed=0)
X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))
     for g in circ.logical_gates]
orc = gf.ChebyshevOracle(spec, 0.25)
basis = (np.arange(0, 4096, 97, dtype=np.int64), None)
rep, hv = gf.gradient_and_hvp(circ, orc, X, basis=basis, batch=16)
cols = gf.hessian_vector_products(circ, orc, [X, [2 * x for x in X], [-x for x in X]], basis=basis, batch=16)
specp, circp, rngp = gf.spinful_layer_circuit(6, 4, False, seed=1, parity=True)
Xp = [gf.manifold.project_tangent_gate(g.matrix, rngp.normal(size=(4, 4)) + 1j * rngp.normal(size=(4, 4)), True)
      for g in circp.logical_gates]
orcp = gf.ChebyshevOracle(specp, 0.25)
repp, hvp = gf.gradient_and_hvp(circp, orcp, Xp, parity_mode=True, sector=0, basis=(np.arange(0, 2048, 61), None),
                                batch=8)
psi = rng.normal(size=2**12) + 1j * rng.normal(size=2**12)
g = gf.manifold.random_unitary(4, rng)
for t in ((0, 1), (3, 11), (11, 2)):
    gf.apply_gate(psi, gf.Gate(g, t))
    gf.hole_contract(psi, psi, t)
    arr = gf.hole_apply(psi, t)
    gf.apply_gate_to_array(arr, gf.Gate(g, (5, 6)))
    gf.hole_contract_array(psi, arr, (5, 6))
gf.apply_gate_1q(psi, gf.manifold.random_unitary(2, rng), 4)
torch.cuda.synchronize()
want = os.environ.get("GF_EXPECT_LIB")
if want:  # the library this process actually mapped
    assert want in open("/proc/self/maps").read(), want
print("sanitize case ok", repr(rep.value), repr(repp.value), len(cols))
