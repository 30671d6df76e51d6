"""Short C2 driver for `ncu --set full` captures (one GPU, no CUDA graph).

    ncu --set full --clock-control none --import-source on \
        -k regex:"attention_kernel|score_rank|sample_kernel|fit_unit_kernel" \
        -s 4 -c 5 -o gpurun_out/full_r01 python tools/profile_decode.py

Launch order: decode #1 (4 launches, skipped by -s 4), decode #2 (score_rank, sample,
fit, sparse attention), dense decode (1 launch).  L2 is flushed before every call.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_12216_b200 import tactic as T  # noqa: E402
from synth import make_layer  # noqa: E402

G, n, C = 4, 131072, 1024
K, V, q = make_layer(1, 8, G, n, seed=0)
to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
Kd, Vd, qd = to(K), to(V), to(q)
idx = T.build_index(Kd, Vd, C, 10, group_size=G)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty_like(qd)
for _ in range(2):
    flush.fill_(1)
    T.decode(qd, idx, 0.9, out=out)
flush.fill_(1)
T.dense_decode(qd, Kd, Vd, out=out)
torch.cuda.synchronize()
print("ok")
