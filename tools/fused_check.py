"""One-launch cluster decode vs the multi-kernel chain on the same index (GPU).

    python tools/fused_check.py [--c2] [--c3]
Prints, per case: order / J / union / fit agreement and the output difference between the
two paths, and CUDA-graph timings of both (cold L2).  Development aid; the parity tests
(tests/test_gpu_fused.py) are the gate.
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
ap.add_argument("--c2", action="store_true")
ap.add_argument("--c3", action="store_true")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--tlog", action="store_true", help="print the one-launch decode's phase stamps (C2)")
args = ap.parse_args()
if args.tlog:
    os.environ["TACTIC_TLOG"] = "1"
B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

dev = torch.device("cuda", 0)
to = lambda a: torch.from_numpy(a).to(dev).to(torch.bfloat16)  # noqa: E731


def compare(name, qd, index, p):
    T.set_options(index, 0)
    rm = T.decode_debug(qd, index, p)
    T.set_options(index, T.OPT_CLUSTER_DECODE)
    rf = T.decode_debug(qd, index, p)
    om, of = rm["out"].float().cpu().numpy(), rf["out"].float().cpu().numpy()
    same_order = np.array_equal(rm["order"], rf["order"])
    dJ = np.abs(rm["J"].astype(np.int64) - rf["J"]).max()
    du = int((rm["union_mask"] != rf["union_mask"]).sum())
    dfit = np.nanmax(np.abs(rm["fit"] - rf["fit"]) / np.maximum(np.abs(rm["fit"]), 1e-30))
    print(f"{name} p={p}: order equal {same_order}, max |dJ| {dJ}, union diffs {du}, fit max rel {dfit:.2e}, "
          f"out max-abs {np.abs(om - of).max():.2e}, lse max-abs {np.abs(rm['lse'].cpu().numpy() - rf['lse'].cpu().numpy()).max():.2e}, "
          f"cluster {index.info()['select_cluster_size']}")


def timeit(qd, index, p, reps):
    out = torch.empty_like(qd)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for nm, opt in [("multi", 0), ("fused", T.OPT_CLUSTER_DECODE)]:
        T.set_options(index, opt)
        T.decode(qd, index, p, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            T.decode(qd, index, p, out=out)
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[nm] = float(np.median(ts))
    T.set_options(index, 0)
    return res


G = 4
K, V, q = make_layer(1, 2, G, 4096, seed=0)
idx = T.build_index(to(K), to(V), 64, 10, group_size=G)
for p in [0.5, 0.9, 0.99]:
    compare("C1x2", to(q), idx, p)
K, V, q = make_layer(1, 2, G, 32768, seed=1)
idx = T.build_index(to(K), to(V), 256, 10, group_size=G)
for p in [0.5, 0.9]:
    compare("32K", to(q), idx, p)
if args.c2:
    K, V, q = make_layer(1, 8, G, 131072, seed=0)
    idx = T.build_index(to(K), to(V), 1024, 10, group_size=G)
    for p in [0.5, 0.9, 0.95]:
        compare("C2", to(q), idx, p)
    print("C2 timing us (graph, cold L2):", timeit(to(q), idx, 0.9, args.reps))
    if args.tlog:
        names = ["start", "scored", "runs exchanged", "ranked", "sampled", "fitted", "lists", "attended", "merged"]
        for _ in range(3):
            torch.cuda.synchronize()
            T.decode(to(q), idx, 0.9)
            torch.cuda.synchronize()
            full = idx.debug_timing().astype(np.int64)
            tl = full[3000:3009]
            print("  CTA(0,0) phases us:", "  ".join(f"{nm} {(t - tl[0]) / 1e3:.2f}" for nm, t in zip(names, tl)))
            sm = full[3010:3014]
            print(f"    sample: first issue {(sm[0] - tl[0]) / 1e3:.2f}, stages {sm[1]}, first consumed "
                  f"{(sm[2] - tl[0]) / 1e3:.2f}, last {(sm[3] - tl[0]) / 1e3:.2f}")
if args.c3:
    K, V, q = make_layer(64, 8, G, 32768, seed=9000)
    idx = T.build_index(to(K), to(V), 256, 10, group_size=G)
    compare("C3", to(q), idx, 0.9)
    print("C3 timing us (graph, cold L2):", timeit(to(q), idx, 0.9, 10))
