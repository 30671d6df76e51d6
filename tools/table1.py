"""Table-1 diagnostics on the GPU (§5.3).

Per (unit, query head) and target p, from the exact score of every clustered token
(tactic_exact_logits, layout order) and the selection the library made (decode_debug):
  Optimal          minimal number of tokens, in descending true score, reaching p
  Cluster-Optimal  minimal prefix of clusters in criticality order reaching p, in tokens
  Tactic           tokens of the head's own selected clusters S_g; and of the GQA union U
  achieved         true cumulative score p(S_g) and p(U) (Eq. 5)
  success          achieved >= p
Budgets are reported as fractions of n.  Measurement tooling: the reductions (softmax,
sort, cumulative sums) use torch on the GPU, the scores and selections come from the
library's kernels; the definitions follow oracle.optimal_budget / cluster_optimal_budget /
cumulative_score, which tests/test_gpu_parity.py checks this module against.

    python tools/table1.py [--layers 2] [--p 0.5 0.9]
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def table1_stats(T, q: torch.Tensor, index, sizes: np.ndarray, ps) -> dict:
    """sizes: int [units][C] cluster sizes (layout: clusters in id order)."""
    dev = q.device
    U, G, n = index.units, index.G, index.n
    L = T.exact_logits(q, index).double()                    # [U][G][n], layout order
    P = torch.softmax(L, dim=-1)
    ps_sorted = torch.sort(P, dim=-1, descending=True).values
    csum_sorted = torch.cumsum(ps_sorted, dim=-1)
    sz = torch.from_numpy(np.asarray(sizes, dtype=np.int64)).to(dev)           # [U][C]
    off = torch.cat([torch.zeros((U, 1), dtype=torch.int64, device=dev), torch.cumsum(sz, dim=1)], dim=1)
    cl = torch.cumsum(P, dim=-1)
    cl = torch.cat([torch.zeros((U, G, 1), dtype=cl.dtype, device=dev), cl], dim=-1)   # cl[k] = sum_{i<k}
    mass = cl.gather(2, off[:, None, 1:].expand(U, G, -1)) - cl.gather(2, off[:, None, :-1].expand(U, G, -1))
    out = {}
    for p in ps:
        dbg = T.decode_debug(q, index, p)
        order = torch.from_numpy(dbg["order"].astype(np.int64)).to(dev)         # [U][G][C]
        J = torch.from_numpy(dbg["J"].astype(np.int64)).to(dev)                 # [U][G]
        umask = torch.from_numpy(dbg["union_mask"].astype(bool)).to(dev)       # [U][C]
        tot = csum_sorted[..., -1:]
        optimal = ((csum_sorted < p * tot).sum(-1) + 1).double()
        m_ord = mass.gather(2, order)
        s_ord = sz[:, None, :].expand(U, G, -1).gather(2, order)
        cm = torch.cumsum(m_ord, dim=-1)
        jco = (cm < p * cm[..., -1:]).sum(-1) + 1
        cs = torch.cumsum(s_ord, dim=-1)
        co = cs.gather(2, (jco - 1)[..., None])[..., 0].double()
        rank = torch.arange(order.shape[-1], device=dev)[None, None, :]
        sel = (rank < J[..., None]).double()
        tac = (cs.double() * 0 + s_ord.double() * sel).sum(-1)
        ach = (m_ord * sel).sum(-1)
        un_tok = (sz.double() * umask.double()).sum(-1)
        un_ach = (mass * umask[:, None, :].double()).sum(-1)                      # [U][G]
        out[str(p)] = {
            "optimal_frac": float(optimal.mean() / n), "cluster_optimal_frac": float(co.mean() / n),
            "tactic_own_frac": float(tac.mean() / n), "tactic_union_frac": float(un_tok.mean() / n),
            "achieved_own": float(ach.mean()), "achieved_union": float(un_ach.mean()),
            "success_own": float((ach >= p).double().mean()), "success_union": float((un_ach >= p).double().mean()),
            "instances": int(U * G),
            "_per_head": {"optimal": optimal.cpu().numpy(), "cluster_optimal": co.cpu().numpy(),
                          "tactic_own": tac.cpu().numpy(), "achieved_own": ach.cpu().numpy(),
                          "achieved_union": un_ach.cpu().numpy()},
        }
    return out


def _cluster_mass(T, q, index, sizes):
    """true softmax mass of every cluster for every head: [U][G][C] (float64, GPU)."""
    dev = q.device
    U, G = index.units, index.G
    P = torch.softmax(T.exact_logits(q, index).double(), dim=-1)
    sz = torch.from_numpy(np.asarray(sizes, dtype=np.int64)).to(dev)
    off = torch.cat([torch.zeros((U, 1), dtype=torch.int64, device=dev), torch.cumsum(sz, dim=1)], dim=1)
    cl = torch.cat([torch.zeros((U, G, 1), dtype=P.dtype, device=dev), torch.cumsum(P, dim=-1)], dim=-1)
    return cl.gather(2, off[:, None, 1:].expand(U, G, -1)) - cl.gather(2, off[:, None, :-1].expand(U, G, -1)), sz


def fig5_variance(T, q, index, sizes, K, V, p: float = 0.9) -> dict:
    """Fig. 5 / P:253 on this data: the threshold rule (Tactic, own-set attention per head)
    against a Quest-like fixed budget with the SAME mean token count per head.  Per head:
    tokens, achieved cumulative score p(I) (Eq. 5) and attention distance
    eps(I) = |o_full - o_I| (Eq. 4, own-set normalisation)."""
    dev = q.device
    U, G = index.units, index.G
    mass, sz = _cluster_mass(T, q, index, sizes)
    o_full = T.dense_decode(q, K, V).float().view(U, G, -1)

    def stats(J, o_sel, order):
        rank = torch.arange(order.shape[-1], device=dev)[None, None, :]
        sel = (rank < torch.from_numpy(J.astype(np.int64)).to(dev)[..., None]).double()
        tok = (sz[:, None, :].expand(U, G, -1).gather(2, order).double() * sel).sum(-1)
        ach = (mass.gather(2, order) * sel).sum(-1)
        eps = torch.linalg.norm(o_full - o_sel.float().view(U, G, -1), dim=-1).double()
        f = lambda x: {"mean": float(x.mean()), "std": float(x.std()), "min": float(x.min()),  # noqa: E731
                       "max": float(x.max())}
        return {"tokens": f(tok), "achieved_p": f(ach), "eps": f(eps)}, tok

    dbg = T.decode_debug(q, index, p)
    order = torch.from_numpy(dbg["order"].astype(np.int64)).to(dev)
    o_t = T.decode_per_head(q, index, p)
    st_t, tok = stats(dbg["J"], o_t, order)
    budget = max(1, int(round(float(tok.mean()))))
    o_f, Jf = T.decode_fixed_budget(q, index, budget, per_head=True)
    st_f, _ = stats(Jf, o_f, order)   # same criticality order (same q, same index)
    return {"p": p, "fixed_budget_tokens": budget, "tactic": st_t, "fixed_budget": st_f, "heads": int(U * G)}


def public(stats: dict) -> dict:
    return {p: {k: v for k, v in d.items() if not k.startswith("_")} for p, d in stats.items()}


if __name__ == "__main__":
    import argparse
    import json

    import bench
    from paper_2502_12216_b200 import build as B
    B.build()
    from paper_2502_12216_b200 import tactic as T

    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--p", type=float, nargs="+", default=[0.5, 0.9])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for L in bench.make_layers(list(range(a.layers)), dev, [(0, h) for h in range(8)]):
        idx = T.build_index(L["K"], L["V"], 1024, 10, group_size=4)
        ex = idx.export()
        sizes = np.stack([np.bincount(ex["assign"][u], minlength=1024) for u in range(idx.units)])
        print(json.dumps(public(table1_stats(T, L["q"], idx, sizes, a.p))))
