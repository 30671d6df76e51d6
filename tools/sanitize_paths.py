"""Small-size runs of every decode path for compute-sanitizer (tools/sanitize_c1.sh):
the kernel chain (and, with the argument `cluster`, the opt-in one-launch cluster
decode), the sequence-sharded stages, the
recent-token tail (both attention splits), the per-head ablation, the fixed budget and the
windows-exact variant.  Checks only that every call completes; parity lives in tests/."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402
from synth import make_layer  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

CLUSTER = len(sys.argv) > 1 and sys.argv[1] == "cluster"  # also the opt-in one-launch decode

to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(torch.bfloat16)  # noqa: E731
G = 4
K, V, q = make_layer(1, 2, G, 4096, seed=3)
idx = T.build_index(to(K), to(V), 64, 3, group_size=G)
qd = to(q)
T.decode(qd, idx, 0.9)
T.decode_debug(qd, idx, 0.5)
if CLUSTER:
    T.set_options(idx, T.OPT_CLUSTER_DECODE)
    T.decode_debug(qd, idx, 0.9)
    T.decode_fixed_budget(qd, idx, 300)
q_pin = qd.cpu().pin_memory()  # zero-copy host decode (entry kernel reads q, merge writes out)
o_pin = torch.empty_like(q_pin).pin_memory()
T.decode_host(q_pin, idx, 0.9, o_pin)
T.decode_host(q_pin, idx, 0.9, o_pin)
T.set_options(idx, T.OPT_DETERMINISTIC)  # the partial merge by the last CTA
T.decode(qd, idx, 0.9)
T.decode_attention_only(qd * 30, idx, torch.empty_like(qd))  # reference-shift window fallback
T.set_options(idx, 0)
T.decode_attention_only(qd * 30, idx, torch.empty_like(qd))
T.set_options(idx, T.OPT_WINDOWS_EXACT)
T.decode(qd, idx, 0.9)
T.set_options(idx, 0)
T.decode_per_head(qd, idx, 0.9)
T.decode_fixed_budget(qd, idx, 300)
T.decode_fixed_budget(qd, idx, 300, per_head=True)
T.dense_decode(qd, to(K), to(V))
T.set_tail_capacity(idx, 64)
kt, vt, _ = make_layer(1, 2, G, 16, seed=4)
T.append(idx, to(kt[0]), to(vt[0]))
T.decode(qd, idx, 0.9)
# sequence-sharded stages (two shards)
shards = [T.build_index(to(K[:, :, s * 2048:(s + 1) * 2048]), to(V[:, :, s * 2048:(s + 1) * 2048]), 32, 3,
                        group_size=G) for s in range(2)]
lm = torch.stack([T.decode_stage1(qd, st).clone() for st in shards])
gmax = lm.max(dim=0).values
mass = torch.stack([T.decode_stage1b(st, gmax).clone() for st in shards]).sum(dim=0)
parts = [T.decode_stage2(qd, st, 0.9, gmax, mass) for st in shards]
T.lse_merge(torch.stack([p[0] for p in parts]).view(2, -1, 128), torch.stack([p[1] for p in parts]).view(2, -1))
# many units: the global attention split
K3, V3, q3 = make_layer(2, 48, G, 1024, seed=5)
idx3 = T.build_index(to(K3), to(V3), 16, 2, group_size=G)
T.decode(to(q3), idx3, 0.9)
torch.cuda.synchronize()
print("sanitize paths ok")
