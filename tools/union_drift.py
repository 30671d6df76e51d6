"""Generator drift check: the union the ORACLE selects at p = 0.9 on its
own 10-iteration clustering, for every unit of the 8 synthetic C2 layers the bench times
(seeds 0..7, KV heads 0..7; same SplitMix64 init as the GPU build).  Compare with the
GPU's union_frac_per_layer in the bench line: equal means the spread is the recipe's
unit-to-unit variance, not GPU clustering quality.

    python tools/union_drift.py [--layers 8] [--iters 10] [--out profiles/r02_union_drift.json]
Runs on the host cores (numpy float64); ~15 s per unit.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import tactic_oracle as O  # noqa: E402
from synth import make_unit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--units", type=int, default=8)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--p", type=float, default=0.9)
ap.add_argument("--out", default="profiles/r02_union_drift.json")
args = ap.parse_args()
n, C, G = 131072, 1024, 4
res = {"n": n, "C": C, "p": args.p, "iters": args.iters, "layers": []}
for sd in range(args.layers):
    lay = []
    for h in range(args.units):
        t0 = time.time()
        u = make_unit(n, G, seed=sd, b=0, h=h)
        idx, km = O.build_index(u["K"], u["V"], C, args.iters, seed=sd, unit=h)
        r = O.decode_unit(u["q"], idx, args.p)
        own = [int(idx.sizes[hd["S"]].sum()) / n for hd in r["heads"]]
        lay.append({"unit": h, "union_frac": len(r["tokens"]) / n, "own_frac": own,
                    "inertia": km["inertia"], "iters_run": km["iters_run"]})
        print(f"layer {sd} unit {h}: union {len(r['tokens']) / n * 100:.2f}% own "
              + " ".join(f"{x * 100:.2f}%" for x in own) + f"  ({time.time() - t0:.1f}s)", flush=True)
    res["layers"].append({"seed": sd, "units": lay, "union_frac": float(np.mean([x["union_frac"] for x in lay]))})
    print(f"layer {sd}: union {res['layers'][-1]['union_frac'] * 100:.2f}%", flush=True)
    json.dump(res, open(args.out, "w"), indent=1)
res["union_frac_mean"] = float(np.mean([L["union_frac"] for L in res["layers"]]))
json.dump(res, open(args.out, "w"), indent=1)
print(f"mean union over layers: {res['union_frac_mean'] * 100:.2f}%")
