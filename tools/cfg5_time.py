"""cfg5 (3840x2160 single frame, 5 levels, 4 px grid, global PCG): device-resident replay time, 3 x 20 replays.

    python tools/cfg5_time.py [libhwflow_cuda.so]   # on the GPU box
"""
import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1610_07159_b200 import build, synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver
dev = Solver(sys.argv[1] if len(sys.argv) > 1 else build.CUDA_LIB)
lib, h = dev.lib, dev.ctx.h
S = SolveSchedule(levels=5, grid_step=4, pcg_iters=5, subdomain_px=0)
fr = synthetic.uhd_pair(0)[0][None]
dev.solve_batch(fr, EnergyParams(), S, None, outputs=("grid_total",))
st = torch.cuda.ExternalStream(lib.hwf_stream(h))
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.hwf_run_device(h)
    e0.record(st)
    for _ in range(20): lib.hwf_run_device(h)
    e1.record(st); e1.synchronize(); lib.hwf_sync(h, None)
    print(f"cfg5 ms/frame {e0.elapsed_time(e1)/20:.3f}", flush=True)
