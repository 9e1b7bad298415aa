import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2506_23775_b200 as gf
sink = torch.zeros(1, dtype=torch.float64, device='cuda'); st = gf._lib.stream_ptr()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for which in (0, 1, 2):
    fl = np.zeros(1)
    gf._lib.check(gf._lib.lib.gf_peak_fp64(which, 148*4, 64, sink.data_ptr(), fl.ctypes.data, st)); torch.cuda.synchronize()
    best = 0
    for _ in range(3):
        e0.record(); gf._lib.check(gf._lib.lib.gf_peak_fp64(which, 148*4, 2048, sink.data_ptr(), fl.ctypes.data, st)); e1.record(); torch.cuda.synchronize()
        best = max(best, fl[0]/(e0.elapsed_time(e1)*1e-3)/1e12)
    print(which, round(best, 2), 'TFLOP/s')
