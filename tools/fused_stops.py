"""Cumulative cost of the one-launch decode's phases on C2: the kernel timed (CUDA graph,
cold L2) when every CTA leaves after phase k (TACTIC_FUSED_STOP=k, one process per k).
    python tools/fused_stops.py   (spawns itself per k)"""
import os
import subprocess
import sys

if len(sys.argv) == 1:
    here = os.path.abspath(__file__)
    for k in [1, 2, 3, 4, 5, 6, 7, 8, 0]:
        env = dict(os.environ, TACTIC_FUSED_STOP=str(k))
        r = subprocess.run([sys.executable, here, "run"], env=env, capture_output=True, text=True)
        print(f"stop {k}: {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
out = torch.empty_like(qd)
T.decode(qd, idx, 0.9, out=out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    T.decode(qd, idx, 0.9, out=out)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(30):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"{np.median(ts):.2f} us (cluster {idx.info()['select_cluster_size']})")
