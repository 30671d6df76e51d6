"""Where a C2 index build's time goes (GPU): the whole tactic_build_index call bracketed by
CUDA events (what bench.py reports as build.ms), the host wall time of the same call, and a
bare cudaMalloc + cudaFree of the index's arena size (the build's one large allocation).

    python tools/build_timing.py [--layers 4] [--iters 10]
"""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12216_b200 import tactic as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()

dev = torch.device("cuda", 0)
layers = bench.make_layers(list(range(args.layers)), dev, [(0, h) for h in range(8)])
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
T.build_index(layers[0]["K"][:, :1, :8192].contiguous(), layers[0]["V"][:, :1, :8192].contiguous(), 64, 2,
              group_size=4)
torch.cuda.synchronize()
for L in layers:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    idx = T.build_index(L["K"], L["V"], 1024, args.iters, group_size=4, seed=L["seed"])
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    info = idx.info()
    nbytes = info["device_bytes"]
    malloc_ms = float("nan")
    if rt is not None:
        p = ctypes.c_void_p()
        m0 = time.perf_counter()
        rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(nbytes))
        m1 = time.perf_counter()
        rt.cudaFree(p)
        malloc_ms = (m1 - m0) * 1e3
    print(f"seed {L['seed']}: events {e0.elapsed_time(e1):.3f} ms, kernels {info['build_gpu_ms']:.3f} ms, host call {1e3 * (t1 - t0):.3f} ms, "
          f"call+sync {1e3 * (t2 - t0):.3f} ms, arena {nbytes / 2**20:.0f} MiB cudaMalloc {malloc_ms:.3f} ms, "
          f"iters {np.asarray(idx.export()['iters_run']).tolist()}")
    del idx
    torch.cuda.synchronize()
