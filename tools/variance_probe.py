"""Run-to-run variance of the bench step on one box: repeated step timings (CUDA events) in fresh
processes, to size the noise band A/B comparisons must beat."""
import os, sys, time, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_08791_b200 as sp
from paper_2410_08791_b200 import _capi
L, d, rows = 48, 1600, 16384
ex = sp.Executor(L, d, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2), numerics=sp.BF16, trace=0)
W = np.empty((d, d), np.float32); b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data); ex.register_layer(i, W, b)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda(); t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
def run(n=10):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
for _ in range(3): run(1)
print("plain", [round(run(), 3) for _ in range(3)])
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "200"], stdout=subprocess.DEVNULL)
print("with smi", [round(run(), 3) for _ in range(3)])
p.terminate()
print("plain again", [round(run(), 3) for _ in range(3)])
