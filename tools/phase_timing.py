"""Per-phase timing of the fused selection kernel on the C2 workload (TACTIC_TLOG=1).

    python tools/phase_timing.py [--p 0.9] [--units-seed 0]
Prints, per phase boundary, the spread over CTAs of %globaltimer stamps relative to the
earliest kernel start (us).  Debug aid only.
"""
import os
import sys

os.environ["TACTIC_TLOG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402
from synth import make_layer  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

G, n, C = 4, 131072, 1024
K, V, q = make_layer(1, 8, G, n, seed=0)
to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
Kd, Vd, qd = to(K), to(V), to(q)
idx = T.build_index(Kd, Vd, C, 10, group_size=G)
print("cluster size R =", idx.info()["select_cluster_size"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["start", "ph1 done", "sync1", "ph2 done", "ph3 done", "sync2", "ph4 done", "sync4"]
R = idx.info()["select_cluster_size"]
for it in range(3):
    flush.fill_(1)
    torch.cuda.synchronize()
    T.decode(qd, idx, 0.9)
    torch.cuda.synchronize()
    full = idx.debug_timing().astype(np.int64)
    t = full[:, :R, :]
    t0 = t[:, :, 0].min()
    if R <= 8:
        ch = full[0, 8:16, :].reshape(-1, 4)
        for c, row in enumerate(ch):
            if row[0] > 0:
                print(f"  chunk {c:2d}: start {(row[0] - t0) / 1e3:7.2f}  issued +{(row[1] - row[0]) / 1e3:5.2f}"
                      f"  waited +{(row[2] - row[1]) / 1e3:5.2f}  computed +{(row[3] - row[2]) / 1e3:5.2f} us")
    at = full.reshape(-1)[192:192 + 35]
    if at[0] > 0:
        b0 = at[0]
        iss = [(x - b0) / 1e3 for x in at[2:18] if x > 0]
        con = [(x - b0) / 1e3 for x in at[18:34] if x > 0]
        print(f"  attention CTA0: start {(b0 - t0) / 1e3:.2f} us after selection start; end +{(at[34] - b0) / 1e3:.2f}")
        print("   tiles issued at", np.round(iss, 2).tolist())
        print("   tiles consumed at", np.round(con, 2).tolist())
    print(f"--- iteration {it}")
    for k, nm in enumerate(names):
        v = (t[:, :, k] - t0) / 1000.0
        ok = t[:, :, k] > 0
        if ok.any():
            print(f"  {nm:10s} min {v[ok].min():7.2f}  median {np.median(v[ok]):7.2f}  max {v[ok].max():7.2f} us")

# p = 1 through the index (1-D bulk copies of whole clusters from the permuted layout)
# vs the dense baseline (TMA tensor boxes from the caller's layout): same bytes
out = torch.empty_like(qd)
for name, fn in [("p=1 via index (bulk runs)", lambda: T.decode(qd, idx, 1.0, out=out)),
                 ("dense (TMA tensor)", lambda: T.dense_decode(qd, Kd, Vd, out=out))]:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{name}: {np.median(ts) * 1e3:.1f} us  ({2 * 8 * n * 256 / (np.median(ts) * 1e-3) / 1e9:.0f} GB/s)")
