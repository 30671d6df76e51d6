"""Regression pins of the frozen input recipe (tactic-synth-v1): the oracle's
per-head selected clusters / tokens and the GQA union at C1 and one 32K unit, p in
{0.5, 0.8, 0.9}.  Writes tests/golden/recipe_regression.json; calls only oracle/ and synth/.

    python tools/make_recipe_golden.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import tactic_oracle as O  # noqa: E402
from synth import make_unit  # noqa: E402

CASES = [{"name": "C1", "n": 4096, "C": 64, "G": 4, "seed": 0, "h": 0, "iters": 10},
         {"name": "32K", "n": 32768, "C": 256, "G": 4, "seed": 0, "h": 1, "iters": 10}]
PS = [0.5, 0.8, 0.9]


def compute(case):
    u = make_unit(case["n"], case["G"], seed=case["seed"], b=0, h=case["h"])
    idx, km = O.build_index(u["K"], u["V"], case["C"], case["iters"], seed=case["seed"], unit=0)
    out = {"case": case, "inertia": float(km["inertia"]), "p": {}}
    for p in PS:
        r = O.decode_unit(u["q"], idx, p)
        out["p"][str(p)] = {"J": [int(h["J"]) for h in r["heads"]],
                            "own_tokens": [int(idx.sizes[h["S"]].sum()) for h in r["heads"]],
                            "union_clusters": int(len(r["U"])), "union_tokens": int(len(r["tokens"]))}
    return out


if __name__ == "__main__":
    res = {"recipe": "tactic-synth-v1", "written_by": "tools/make_recipe_golden.py (oracle/ + synth/ only)",
           "cases": [compute(c) for c in CASES]}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        "recipe_regression.json")
    json.dump(res, open(path, "w"), indent=1)
    for c in res["cases"]:
        print(c["case"]["name"], {p: (v["own_tokens"], v["union_tokens"]) for p, v in c["p"].items()})
