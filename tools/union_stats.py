"""Per-unit selected fractions on the C2 workload (GPU index build, decode_debug): the
share of tokens in each unit's GQA union and in each head's own selection.

    python tools/union_stats.py [--p 0.9] [--seed 0] [--iters 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402
from synth import make_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=float, default=0.9)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--iters", type=int, default=10)
args = ap.parse_args()
B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

G, n, C = 4, 131072, 1024
K, V, q = make_layer(1, 8, G, n, seed=args.seed)
to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
Kd, Vd, qd = to(K), to(V), to(q)
idx = T.build_index(Kd, Vd, C, args.iters, group_size=G)
ex = idx.export()
res = T.decode_debug(qd, idx, args.p)
sizes = np.stack([np.bincount(ex["assign"][u], minlength=C) for u in range(8)])
for u in range(8):
    um = res["union_mask"][u].astype(bool)
    own = []
    for g in range(G):
        J = int(res["J"][u, g])
        own.append(sizes[u][res["order"][u, g, :J]].sum() / n)
    print(f"unit {u}: union {sizes[u][um].sum() / n * 100:5.2f}%  own " +
          " ".join(f"{x * 100:5.2f}%" for x in own) + f"  iters {ex['iters_run'][u]}  empty {int((sizes[u] == 0).sum())}")
tot = sum(sizes[u][res["union_mask"][u].astype(bool)].sum() for u in range(8))
print(f"all units: union {tot / (8 * n) * 100:.2f}% of tokens")
