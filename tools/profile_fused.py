"""One C2 decode step through the one-launch cluster decode (for ncu):
    ncu --set full -k regex:decode_fused -s 2 -c 1 python tools/profile_fused.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402
from synth import make_layer  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
K, V, q = make_layer(1, 8, 4, 131072, seed=0)
idx = T.build_index(to(K), to(V), 1024, 10, group_size=4)
T.set_options(idx, T.OPT_CLUSTER_DECODE)
qd = to(q)
for _ in range(4):
    T.decode(qd, idx, 0.9)
torch.cuda.synchronize()
print("cluster size", idx.info()["select_cluster_size"])
