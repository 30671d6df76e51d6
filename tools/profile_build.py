"""C2 index-build driver for ncu captures of the tcgen05 k-means assignment GEMM (B2).

    ncu --set full -k regex:km_assign_tc -s 3 -c 1 -o gpurun_out/km python tools/profile_build.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12216_b200 import tactic as T  # noqa: E402

dev = torch.device("cuda", 0)
L = bench.make_layers([0], dev, [(0, h) for h in range(8)])[0]
idx = T.build_index(L["K"], L["V"], 1024, 4, group_size=4)
ex = idx.export()  # (runs the inertia kernel)
torch.cuda.synchronize()
print("ok", idx.info()["units"])
