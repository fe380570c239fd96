import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2603_00035_b200 as rfk
from paper_2603_00035_b200 import workload as wl
for n in (256, 1024, 4096):
    F = wl.randers_fields(n, 1, 0.2)
    src = wl.point_source(n, n)
    T64, r64 = rfk.solve(*F, src, 1.0 / n)
    T32, r32 = rfk.solve_f32(*F, src, 1.0 / n, max_iters=50)
    d = (T32.double() - T64).abs()
    i = int(d.argmax()); r, c = divmod(i, n)
    print(f"n={n} K64={r64.iterations} K32={r32.iterations} hist32={['%.1e'%x for x in r32.max_delta_history[-4:]]}")
    print(f"   max abs {d.max().item():.3e} at ({r},{c}) T64={T64[r,c].item():.6f} T32={T32[r,c].item():.6f}; mean abs {d.mean().item():.3e}; max T {T64.max().item():.3f}")
    big = T64 > 0.05
    print(f"   max rel (T>0.05) {(d[big] / T64[big]).max().item():.3e}")
    # fp32 rounding of the fp64 solution itself, as a floor
    print(f"   rounding floor {((T64.float().double() - T64).abs()).max().item():.3e}")
