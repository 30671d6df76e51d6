"""In-kernel %globaltimer stamps of the decode kernels on the C2 workload (TACTIC_TLOG=1).

    python tools/phase_timing.py [--select fused|multi]
Debug aid only: prints the fit-kernel phases (multi path) or the fused-kernel phases,
and CTA 0 of the attention kernel (tiles issued / consumed), relative times in us.
"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--select", default="multi")
args = ap.parse_args()
os.environ["TACTIC_TLOG"] = "1"
os.environ["TACTIC_SELECT"] = args.select
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
R = idx.info()["select_cluster_size"]
print("select cluster size R =", R)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty_like(qd)
for it in range(4):
    flush.fill_(1)
    torch.cuda.synchronize()
    T.decode(qd, idx, 0.9, out=out)
    torch.cuda.synchronize()
    full = idx.debug_timing().astype(np.int64).reshape(-1)
    if it < 2:
        continue
    print(f"--- iteration {it}")
    if R == 0:
        fs = full[256:256 + 32].reshape(4, 8)
        last = full[256 + 64 + 8:256 + 64 + 12]
        t0 = fs[:, 0][fs[:, 0] > 0].min()
        names = ["start", "pdl_wait", "staged", "fit", "k*", "J+mark"]
        cl = full[256 + 96:256 + 128].reshape(4, 8)
        for h in range(4):
            print(f"  fit u0 g{h}: " + "  ".join(f"{nm} {(fs[h, i] - t0) / 1e3:6.2f}" for i, nm in enumerate(names)))
            print(f"     SM clock over the CTA: {(cl[h, 5] - cl[h, 0]) / max(fs[h, 5] - fs[h, 0], 1) * 1e3:.0f} MHz")
        print("  last head compaction: start %.2f end %.2f; last unit prefix: start %.2f end %.2f" %
              tuple((x - t0) / 1e3 if x > 0 else float("nan") for x in last))
    else:
        t = full.reshape(-1, 16, 8)[:, :R, :]
        t0 = t[:, :, 0].min()
        names = ["start", "ph1 done", "sync1", "ph2 done", "ph3 done", "sync2", "ph4 done", "sync4"]
        for k, nm in enumerate(names):
            v = (t[:, :, k] - t0) / 1000.0
            ok = t[:, :, k] > 0
            if ok.any():
                print(f"  {nm:10s} min {v[ok].min():7.2f}  median {np.median(v[ok]):7.2f}  max {v[ok].max():7.2f} us")
    at = full[192:192 + 35]
    if at[0] > 0:
        b0 = at[0]
        iss = [(x - b0) / 1e3 for x in at[2:18] if x > 0]
        con = [(x - b0) / 1e3 for x in at[18:34] if x > 0]
        print(f"  attention CTA0: starts {(b0 - t0) / 1e3:.2f} us after selection start; ends +{(at[34] - b0) / 1e3:.2f}")
        print("   tiles issued at", np.round(iss, 2).tolist())
        print("   tiles consumed at", np.round(con, 2).tolist())
