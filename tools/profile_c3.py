"""C3 (batch 64, 32K, 512 units, C = 256) decode driver for ncu launch lists / captures.

    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score_rank|sample|fit|attention" \
        --csv --log-file gpurun_out/c3_launches.csv python tools/profile_c3.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12216_b200 import tactic as T  # noqa: E402

dev = torch.device("cuda", 0)
L = bench.make_layers([9000], dev, [(b, h) for b in range(64) for h in range(8)], n=32768)[0]
idx = T.build_index(L["K"], L["V"], 256, 10, group_size=4, seed=9000)
out = torch.empty_like(L["q"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    flush.fill_(1)
    T.decode(L["q"], idx, 0.9, out=out)
flush.fill_(1)
T.dense_decode(L["q"], L["K"], L["V"], out=out)
torch.cuda.synchronize()
print("ok")
