mkdir -p gpurun_out/r26
for i in 1 2; do timeout 300 python bench_configs.py --one c1 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['full_sum_grad_hvp_s'], d['trust_region_5_iterations_s'])"; done
python - <<'PY'
import time, torch, numpy as np
import paper_2506_23775_b200 as gf
spec, circ, rng = gf.spinful_layer_circuit(4, 3, False, seed=0)
X = [gf.manifold.project_tangent_gate(g.matrix, rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)), False) for g in circ.logical_gates]
orc = gf.DenseOracle(spec, 0.25)
for _ in range(5): gf.gradient_and_hvp(circ, orc, X)
torch.cuda.synchronize()
ts=[]
for _ in range(20):
    t0=time.perf_counter(); rep,hv=gf.gradient_and_hvp(circ, orc, X); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
print('per-call ms', [round(t*1e3,3) for t in ts])
print(rep.engine)
import cProfile, pstats
pr=cProfile.Profile(); pr.enable()
for _ in range(50): gf.gradient_and_hvp(circ, orc, X)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats('cumtime').print_stats(18)
PY
