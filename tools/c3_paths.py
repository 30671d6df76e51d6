"""C3 (batch 64 x 8 KV heads, 32K tokens, C = 256, p = 0.9): the kernel chain vs the
one-launch cluster decode (TACTIC_OPT_CLUSTER_DECODE) on the same index, CUDA graph,
cold L2, plus their agreement."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_12216_b200 import build as B  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

dev = torch.device("cuda", 0)
L = bench.make_layers([9000], dev, [(b, h) for b in range(64) for h in range(8)], n=32768)[0]
idx = T.build_index(L["K"], L["V"], 256, 10, group_size=4, seed=9000)
q = L["q"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
outs = {}
for nm, opt in [("chain", 0), ("cluster", T.OPT_CLUSTER_DECODE)]:
    T.set_options(idx, opt)
    out = torch.empty_like(q)
    T.decode(q, idx, 0.9, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        T.decode(q, idx, 0.9, out=out)
    ts = []
    for _ in range(10):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    res[nm] = float(np.median(ts))
    outs[nm] = out.float().clone()
    print(nm, f"{res[nm]:.1f} us", "cluster size", idx.info()["select_cluster_size"], flush=True)
d = (outs["chain"] - outs["cluster"]).abs().max().item()
print("max |chain - cluster| =", d)
