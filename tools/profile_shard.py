"""C4 shard (131072 tokens x 8 KV heads, C = 1024) sequence-sharded stages, for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12216_b200 import tactic as T  # noqa: E402

dev = torch.device("cuda", 0)
L = bench.make_layers([0], dev, [(0, h) for h in range(8)])[0]
idx = T.build_index(L["K"], L["V"], 1024, 10, group_size=4)
for _ in range(3):
    lm = T.decode_stage1(L["q"], idx)
    ms = T.decode_stage1b(idx, lm)
    o, l = T.decode_stage2(L["q"], idx, 0.9, lm, ms)
    out = T.lse_merge(o.view(1, -1, 128), l.view(1, -1))
torch.cuda.synchronize()
print("ok")
