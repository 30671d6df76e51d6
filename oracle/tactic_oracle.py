"""Tactic CPU float64 ORACLE -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.  The
product path (`paper_2502_12216_b200/`, `csrc/`) never imports it and shares no
code, header, table or constant generator with it.

What it computes: the decode-time sparse attention of
"Tactic: Adaptive Sparse Attention with Clustering and Distribution Fitting for
Long-Context LLMs" (arXiv 2502.12216), written as a plain, slow, step-by-step
numpy float64 program in the paper's order and notation.  Citations `P:n` are
lines of /root/reference/PAPER.md; `S:n` lines of SPEC.md (interfaces only);
"reading k" refers to DESIGN.md §"Readings of the paper" (the numbered list).

Inputs are the generator's bf16 tensors (float32 arrays holding bf16 values),
widened exactly to float64.  Centroids handed to decode are in the index
storage format: float32 (reading 18), i.e. `float32(c)` of the exact member
mean `c`.

Pins (tests/test_oracle_*.py): library k-means (scikit-learn Lloyd, same init),
brute-force subsets for the optimal selection, closed forms (harmonic sums,
two-point fit), full attention via torch SDPA / scipy, the Appendix-A bound,
LSE-merge identities, SPEC worked examples (tests/golden/).
Parity unpinned: the accuracy of the estimated total mass W on any real model
distribution (the paper prints no worked example of Alg. 1); see DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# B1. Initialisation sampler (§4.2 "randomly sampling SeqLen / Average
# cluster size data points as the initial cluster centroids"; footnote: no
# k-means++).  Reading 3: uniform without replacement via SplitMix64 + partial
# Fisher-Yates, seeded with seed + (unit+1)*0x9E3779B97F4A7C15 (mod 2^64).
# The library implements the same counter-based generator independently.
# ---------------------------------------------------------------------------
def _splitmix64_stream(state: int):
    while True:
        state = (state + SPLITMIX_GAMMA) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def init_indices(n: int, C: int, seed: int, unit: int) -> np.ndarray:
    """C distinct token indices in [0, n) (the initial centroids' tokens)."""
    if not (1 <= C <= n):
        raise ValueError("need 1 <= C <= n (S:115)")
    gen = _splitmix64_stream((seed + (unit + 1) * SPLITMIX_GAMMA) & MASK64)
    a: Dict[int, int] = {}
    out = np.empty(C, dtype=np.int64)
    for j in range(C):
        r = j + next(gen) % (n - j)
        aj, ar = a.get(j, j), a.get(r, r)
        a[j], a[r] = ar, aj
        out[j] = ar
    return out


# ---------------------------------------------------------------------------
# B2-B4. K-means (§4.2; max 10 iterations P:402 §5.1).
# Reading 4: "distance" = squared Euclidean; reading 5: convergence = exact
# assignment fixpoint; reading 6: an empty cluster keeps its previous
# centroid; reading 7: ties -> lowest cluster id.
# ---------------------------------------------------------------------------
def _sq_dist_argmin(K: np.ndarray, c: np.ndarray, block: int = 4096):
    """argmin_j sum_d (K_i - c_j)^2 with ties to the lowest j, and the min value.
    The squared distance is expanded as |k|^2 - 2 k.c + |c|^2 (a library matmul),
    evaluated in float64 over token blocks (blocking only bounds memory)."""
    n = K.shape[0]
    cn = np.einsum("jd,jd->j", c, c)
    assign = np.empty(n, dtype=np.int64)
    mind = np.empty(n, dtype=np.float64)
    for s in range(0, n, block):
        kb = K[s:s + block]
        kn = np.einsum("id,id->i", kb, kb)
        dist = kn[:, None] - 2.0 * (kb @ c.T) + cn[None, :]
        a = np.argmin(dist, axis=1)  # first minimum -> lowest id
        assign[s:s + block] = a
        mind[s:s + block] = dist[np.arange(len(a)), a]
    return assign, mind


def kmeans(K: np.ndarray, C: int, iters: int = 10, init: Optional[np.ndarray] = None,
           seed: int = 0, unit: int = 0) -> dict:
    """Lloyd's algorithm exactly as §4.2 describes it (O1-O3 of DESIGN.md).

    O1  c^0_j = K[init_j]
    O2  for t = 1..T: a_t(i) = argmin_j |K_i - c^{t-1}_j|^2 ; c^t_j = mean{K_i : a_t(i)=j}
        (c^{t-1}_j kept if empty); stop when t >= 2 and a_t == a_{t-1}.
    O3  outputs a = a_t, c = c^t, inertia = sum_i |K_i - c_{a(i)}|^2, iterations used.
    """
    K = np.asarray(K, dtype=np.float64)
    n, d = K.shape
    if iters < 1:
        raise ValueError("iters must be >= 1")
    if init is None:
        init = init_indices(n, C, seed, unit)
    init = np.asarray(init, dtype=np.int64)
    if init.shape != (C,) or init.min() < 0 or init.max() >= n:
        raise ValueError("init must hold C token indices in [0, n)")
    c = K[init].copy()
    prev = None
    inertia_trace: List[float] = []
    t_used = 0
    for t in range(1, iters + 1):
        a, _ = _sq_dist_argmin(K, c)
        sums = np.zeros((C, d))
        np.add.at(sums, a, K)
        cnt = np.bincount(a, minlength=C)
        nz = cnt > 0
        c_new = c.copy()
        c_new[nz] = sums[nz] / cnt[nz, None]
        c = c_new
        t_used = t
        inertia_trace.append(float(np.sum((K - c[a]) ** 2)))
        if prev is not None and np.array_equal(a, prev):
            break
        prev = a
    inertia = float(np.sum((K - c[a]) ** 2))
    return {"assign": a, "centroids": c, "inertia": inertia, "iters_run": t_used,
            "sizes": np.bincount(a, minlength=C), "inertia_trace": inertia_trace}


def layout_from_assign(assign: np.ndarray, C: int):
    """O4 / B5: clusters in id order, tokens inside a cluster in ascending original
    index.  Returns offsets [C+1] and perm [n] (original token ids)."""
    assign = np.asarray(assign, dtype=np.int64)
    perm = np.argsort(assign, kind="stable")
    sizes = np.bincount(assign, minlength=C)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return offsets, perm


@dataclass
class Index:
    """One unit's index: original K/V (f64), assignment, storage-format centroids."""
    K: np.ndarray
    V: np.ndarray
    assign: np.ndarray
    centroids: np.ndarray          # float64 values of the float32 storage format
    offsets: np.ndarray
    perm: np.ndarray
    sizes: np.ndarray
    C: int

    @property
    def n(self) -> int:
        return self.K.shape[0]


def make_index(K, V, centroids, assign) -> Index:
    """Index from a given clustering; centroids are rounded to the float32 storage
    format (reading 18), exactly as tactic_index_import does."""
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    cs = np.asarray(centroids, dtype=np.float64).astype(np.float32).astype(np.float64)
    C = cs.shape[0]
    assign = np.asarray(assign, dtype=np.int64)
    offsets, perm = layout_from_assign(assign, C)
    return Index(K, V, assign, cs, offsets, perm, np.diff(offsets), C)


def build_index(K, V, C: int, iters: int = 10, init=None, seed: int = 0, unit: int = 0):
    km = kmeans(K, C, iters, init=init, seed=seed, unit=unit)
    return make_index(K, V, km["centroids"], km["assign"]), km


# ---------------------------------------------------------------------------
# Decode (per unit, per query head).  §4.3 querying, §4.4 fitting (Alg. 1,
# P:747-766), §4.5 GQA union, §4.6 attention on selected tokens.
# ---------------------------------------------------------------------------
DEFAULT_SAMPLING = {"exact_frac": 0.02, "p1": 0.10, "p2": 0.60, "window_half_frac": 0.0025}


def _ppm(f: float) -> int:
    """A sampling fraction quantised to parts per million (round half up): the
    integer the rule below works with, so that every party derives the same N, x1,
    x2, w from the same fractions whatever their floating-point width."""
    return int(np.floor(float(f) * 1e6 + 0.5))


def sample_constants(n: int, exact_frac: float = 0.02, p1: float = 0.10, p2: float = 0.60,
                     window_half_frac: float = 0.0025) -> dict:
    """O6: integer N (exact head), window centres x1, x2 and half-width w.

    P:376: the first N = "1-2% of total tokens" ranks are exact (reading 10: the upper
    end, exact_frac = 0.02).  P:373: the windows sit at "e.g., 10% and 60%" of the
    sorted tokens (p1, p2).  Reading 8: the window half-width is a fraction of n
    (window_half_frac = 0.25%).  With e, q1, q2, h the fractions in ppm:
        N  = ceil(e n / 1e6),   x_k = round_half_up(q_k n / 1e6),
        w  = max(1, round_half_up(h n / 1e6)).
    fallback = exact weights for every rank when the windows collide with the head,
    with each other or with the end (tiny n)."""
    e, q1, q2, h = _ppm(exact_frac), _ppm(p1), _ppm(p2), _ppm(window_half_frac)
    if not (e >= 1 and h >= 1 and 1 <= q1 < q2 < 1000000):
        raise ValueError("need exact_frac, window_half_frac > 0 and 0 < p1 < p2 < 1")
    N = (e * n + 999999) // 1000000
    x1 = (2 * q1 * n + 1000000) // 2000000
    x2 = (2 * q2 * n + 1000000) // 2000000
    w = max(1, (2 * h * n + 1000000) // 2000000)
    fallback = (x1 - w <= N) or (x1 + w >= x2 - w) or (x2 + w > n)
    return {"N": N, "x1": x1, "x2": x2, "w": w, "fallback": bool(fallback)}


def criticality(q_g: np.ndarray, idx: Index) -> np.ndarray:
    """§4.3: criticality of each cluster = dot product of q and the centroid
    (no 1/sqrt(d): monotone)."""
    return idx.centroids @ np.asarray(q_g, dtype=np.float64)


def sort_clusters(crit: np.ndarray) -> np.ndarray:
    """Order pi: descending criticality, ties -> lower cluster id."""
    C = crit.shape[0]
    return np.lexsort((np.arange(C), -crit))


def sorted_tokens(idx: Index, order: np.ndarray) -> np.ndarray:
    """The 'partially sorted token list' of P:368: clusters in order pi, tokens of a
    cluster in ascending original index."""
    return np.concatenate([idx.perm[idx.offsets[j]:idx.offsets[j + 1]] for j in order]) \
        if len(order) else np.zeros(0, dtype=np.int64)


def fit_two_point(x1: float, mu1: float, x2: float, mu2: float):
    """O8: solve y = a/x + b through (x1, mu1), (x2, mu2) (Alg. 1 l.4)."""
    a = (mu1 - mu2) * x1 * x2 / (x2 - x1)
    b = mu1 - a / x1
    return a, b


def token_budget(w: np.ndarray, P: float) -> int:
    """Alg. 1 l.10: minimal k with sum_{i<=k} w_i >= P * sum_i w_i (1-based)."""
    cum = np.cumsum(np.asarray(w, dtype=np.float64))
    W = cum[-1]
    return int(np.argmax(cum >= P * W)) + 1


def decode_head(q_g: np.ndarray, idx: Index, p: float, windows_exact: bool = False,
                sampling: Optional[dict] = None) -> dict:
    """Per query head: O5-O10 (selection) for one unit.  Returns the order pi, the
    per-cluster end ranks, the fit and the selected cluster set S_g.
    windows_exact: SPEC's variant -- the window ranks keep their exact
    weights too ("exact values taking precedence"); default reading 11: only i <= N.
    sampling: the fractions of sample_constants (default DEFAULT_SAMPLING)."""
    n, C = idx.n, idx.C
    d = idx.K.shape[1]
    q_g = np.asarray(q_g, dtype=np.float64)
    crit = criticality(q_g, idx)
    order = sort_clusters(crit)
    sizes_sorted = idx.sizes[order]
    ends = np.cumsum(sizes_sorted)                 # e_r, r = 1..C (1-based ranks)
    starts = ends - sizes_sorted                   # s_r
    tok = sorted_tokens(idx, order)                # tau(i) = tok[i-1]
    sc = sample_constants(n, **(sampling or {}))
    N, x1, x2, w = sc["N"], sc["x1"], sc["x2"], sc["w"]
    scale = 1.0 / np.sqrt(d)

    def logit(ranks):  # O7: l_i = q . K_tau(i) / sqrt(d), ranks 1-based
        return (idx.K[tok[np.asarray(ranks) - 1]] @ q_g) * scale

    out = {"crit": crit, "order": order, "ends": ends, "starts": starts, **sc}
    if sc["fallback"]:
        # reading (O6): exact weights for every rank (cluster-optimal), S:255 analogue
        ranks = np.arange(1, n + 1)
        ell = logit(ranks)
        m = float(ell.max())
        what = np.exp(ell - m)
        a = b = mu1 = mu2 = float("nan")
    else:
        head = np.arange(1, N + 1)
        win1 = np.arange(x1 - w, x1 + w + 1)
        win2 = np.arange(x2 - w, x2 + w + 1)
        l_head, l_w1, l_w2 = logit(head), logit(win1), logit(win2)
        m = float(max(l_head.max(), l_w1.max(), l_w2.max()))      # shift (reading 13)
        e_head = np.exp(l_head - m)                                # Alg.1 l.9, i <= N
        mu1 = float(np.mean(np.exp(l_w1 - m)))                     # Alg.1 l.4
        mu2 = float(np.mean(np.exp(l_w2 - m)))
        a, b = fit_two_point(float(x1), mu1, float(x2), mu2)       # O8
        i = np.arange(N + 1, n + 1, dtype=np.float64)
        what = np.concatenate([e_head, np.maximum(0.0, a / i + b)])  # Alg.1 l.10 + reading 12
        if windows_exact:
            what[win1 - 1] = np.exp(l_w1 - m)
            what[win2 - 1] = np.exp(l_w2 - m)
    cum0 = np.concatenate([[0.0], np.cumsum(what)])                # cum(k), k = 0..n
    W = float(cum0[n])
    cum_end = cum0[ends]
    if p >= 1.0:
        J = C                                                      # reading 15
    else:
        J = int(np.argmax(cum_end >= p * W)) + 1                   # O10
    sel_pos = np.arange(J)
    S_g = np.sort(order[sel_pos][sizes_sorted[sel_pos] > 0])
    out.update({"m": m, "mu1": mu1, "mu2": mu2, "a": a, "b": b, "W": W, "J": J,
                "cum_end": cum_end, "S": S_g, "what": what,
                "phat": float(cum_end[J - 1] / W) if W > 0 else float("nan")})
    return out


def full_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray):
    """Eq. 1 / Eq. 2 read as softmax(q K^T / sqrt(d)) V
    (reading 1).  Returns o [G][d] and natural-log LSE [G]."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    ell = (q @ K.T) / np.sqrt(K.shape[1])
    m = ell.max(axis=1, keepdims=True)
    e = np.exp(ell - m)
    s = e.sum(axis=1, keepdims=True)
    return (e @ V) / s, (m + np.log(s))[:, 0]


def sparse_attention(q, K, V, I):
    """Eq. 3: attention renormalised over the index set I."""
    I = np.asarray(I, dtype=np.int64)
    if I.size == 0:
        raise ValueError("empty index set (S:344)")
    return full_attention(q, np.asarray(K)[I], np.asarray(V)[I])


def cluster_tokens(idx: Index, clusters) -> np.ndarray:
    clusters = np.asarray(clusters, dtype=np.int64)
    if clusters.size == 0:
        return np.zeros(0, dtype=np.int64)
    return np.sort(np.concatenate([idx.perm[idx.offsets[j]:idx.offsets[j + 1]] for j in clusters]))


def decode_unit(q: np.ndarray, idx: Index, p: float, windows_exact: bool = False,
                sampling: Optional[dict] = None) -> dict:
    """O5-O12 for one unit and its G query heads: per-head selection, GQA union
    U = union_g S_g (§4.5), attention of every head over U (reading 17)."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    G = q.shape[0]
    heads = [decode_head(q[g], idx, p, windows_exact, sampling) for g in range(G)]
    mask = np.zeros(idx.C, dtype=bool)
    for h in heads:
        mask[h["S"]] = True
    U = np.nonzero(mask)[0]
    toks = cluster_tokens(idx, U)
    o, lse = sparse_attention(q, idx.K, idx.V, toks)
    return {"heads": heads, "union_mask": mask, "U": U, "tokens": toks, "o": o, "lse": lse}


def fixed_budget_select(q_g: np.ndarray, idx: Index, k: int) -> dict:
    """Quest-like baseline (SPEC fixed_budget_select S:465): clusters in
    criticality order (O5) until the head holds k tokens -- the first cluster whose end
    rank reaches k closes the set (cluster granularity, reading 14)."""
    if not 1 <= k <= idx.n:
        raise ValueError("k out of range")
    order = sort_clusters(criticality(q_g, idx))
    ends = np.cumsum(idx.sizes[order])
    J = int(np.argmax(ends >= k)) + 1
    S = order[:J]
    return {"order": order, "J": J, "S": S[idx.sizes[S] > 0]}


def decode_unit_per_head(q: np.ndarray, idx: Index, p: float) -> dict:
    """Per-head loading (the ablation of P:695; SPEC's own-set normalisation):
    every head attends only the tokens of its own selection S_g (Eq. 3 over S_g)."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    heads = [decode_head(q[g], idx, p) for g in range(q.shape[0])]
    o = np.stack([sparse_attention(q[g], idx.K, idx.V, cluster_tokens(idx, heads[g]["S"]))[0][0]
                  for g in range(q.shape[0])])
    return {"heads": heads, "o": o}


# ---------------------------------------------------------------------------
# Multi-step generation.  P:112 (§1): "performs full
# attention on newly generated tokens" and updates the clustering periodically;
# SPEC assign_token.
# ---------------------------------------------------------------------------
def assign_tokens(K_new: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    """Nearest centroid of each new key: argmin_j |k - c_j|^2 (reading 4), ties to
    the lowest id (reading 7); float64."""
    a, _ = _sq_dist_argmin(np.asarray(K_new, dtype=np.float64), np.asarray(centroids, dtype=np.float64))
    return a


def decode_unit_with_tail(q: np.ndarray, idx: Index, p: float, K_tail: np.ndarray, V_tail: np.ndarray) -> dict:
    """decode_unit's selection over the clustered tokens (O5-O11 unchanged); every head
    then attends the union U plus the whole dense tail of appended tokens (O12 over
    U-tokens + tail)."""
    r = decode_unit(q, idx, p)
    K_tail = np.asarray(K_tail, dtype=np.float64).reshape(-1, idx.K.shape[1])
    V_tail = np.asarray(V_tail, dtype=np.float64).reshape(-1, idx.V.shape[1])
    K_all = np.concatenate([np.asarray(idx.K, dtype=np.float64), K_tail])
    V_all = np.concatenate([np.asarray(idx.V, dtype=np.float64), V_tail])
    toks = np.concatenate([r["tokens"], idx.n + np.arange(K_tail.shape[0])])
    o, lse = sparse_attention(np.atleast_2d(np.asarray(q, dtype=np.float64)), K_all, V_all, toks)
    r.update(o=o, lse=lse, tokens=toks)
    return r


# ---------------------------------------------------------------------------
# Diagnostics (Eq. 4-6, Table 1 methodology) -- test/diagnostic only.
# ---------------------------------------------------------------------------
def exact_scores(q_g, K) -> np.ndarray:
    """s_i of Eq. 2."""
    ell = (np.asarray(K, dtype=np.float64) @ np.asarray(q_g, dtype=np.float64)) / np.sqrt(K.shape[1])
    e = np.exp(ell - ell.max())
    return e / e.sum()


def cumulative_score(q_g, K, I) -> float:
    """p(I) of Eq. 5."""
    return float(exact_scores(q_g, K)[np.asarray(I, dtype=np.int64)].sum())


def attention_distance(q_g, K, V, I) -> float:
    """epsilon(I) of Eq. 4."""
    o, _ = full_attention(q_g, K, V)
    ot, _ = sparse_attention(q_g, K, V, I)
    return float(np.linalg.norm(o[0] - ot[0]))


def distance_bound(q_g, K, V, I) -> float:
    """Eq. 6 / App. A: 2 (1 - p(I)) max_i |v_i|."""
    return 2.0 * (1.0 - cumulative_score(q_g, K, I)) * float(np.max(np.linalg.norm(V, axis=1)))


def optimal_budget(q_g, K, P: float) -> int:
    """descending true attention score until the cumulative score >= P."""
    s = np.sort(exact_scores(q_g, K))[::-1]
    return token_budget(s, P)


def cluster_optimal_budget(q_g, idx: Index, P: float) -> int:
    """Table 1 'Cluster-Optimal': clusters in criticality order, exact
    scores, minimal cluster prefix reaching P (tokens counted)."""
    order = sort_clusters(criticality(q_g, idx))
    s = exact_scores(q_g, idx.K)
    mass = np.array([s[idx.perm[idx.offsets[j]:idx.offsets[j + 1]]].sum() for j in order])
    sizes = idx.sizes[order]
    cum = np.cumsum(mass)
    J = int(np.argmax(cum >= P * cum[-1])) + 1
    return int(sizes[:J].sum())


def lse_merge(o_parts: np.ndarray, lse_parts: np.ndarray):
    """S9: lse = logsumexp_s lse_s ; o = sum_s exp(lse_s - lse) o_s."""
    o_parts = np.asarray(o_parts, dtype=np.float64)
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    mx = np.max(lse_parts, axis=0)
    wts = np.exp(lse_parts - mx)
    tot = wts.sum(axis=0)
    lse = mx + np.log(tot)
    o = np.einsum("s...,s...d->...d", wts / tot, o_parts)
    return o, lse


# ---------------------------------------------------------------------------
# Sequence-sharded mode (a proposed reading, reading 23):
# the paper's global rule "descending criticality until the estimated mass
# reaches P of the estimated total" evaluated over S shard-local fits in
# a common exponent frame on a shared criticality grid.
# ---------------------------------------------------------------------------
SHARD_GRID_T = 512
SHARD_GRID_STEP = 1.0 / 16.0


def shard_stage1(q_g, idx: Index) -> dict:
    """Local S1-S5: local order, local fit; emits (m_s, theta_max_s) with
    theta = crit / sqrt(d)."""
    h = decode_head(q_g, idx, 0.5)   # p irrelevant for the stage-1 quantities
    d = idx.K.shape[1]
    theta = h["crit"] / np.sqrt(d)
    h["theta"] = theta
    h["theta_max"] = float(theta.max())
    return h


def shard_mass_vector(h: dict, m_glob: float, theta_max_glob: float) -> np.ndarray:
    """Stage 1b: [W_s, M_s(theta_t) for t = 1..T] in the global exponent frame.
    M_s(theta) = estimated local mass of clusters with crit/sqrt(d) >= theta."""
    f = np.exp(h["m"] - m_glob)
    what = h["what"] * f
    cum0 = np.concatenate([[0.0], np.cumsum(what)])
    vec = np.empty(SHARD_GRID_T + 1)
    vec[0] = cum0[-1]
    theta_sorted = h["theta"][h["order"]]
    for t in range(1, SHARD_GRID_T + 1):
        th = theta_max_glob - t * SHARD_GRID_STEP
        r = int(np.sum(theta_sorted >= th))       # clusters at or above th: a prefix of pi
        vec[t] = cum0[h["ends"][r - 1]] if r > 0 else 0.0
    return vec


def shard_threshold(total_vec: np.ndarray, p: float, theta_max_glob: float):
    """Stage 2 rule: theta* = largest grid theta_t with sum_s M_s(theta_t) >= p sum_s W_s;
    None means the grid floor was reached (select everything)."""
    if p >= 1.0:
        return None
    W = total_vec[0]
    for t in range(1, SHARD_GRID_T + 1):
        if total_vec[t] >= p * W:
            return theta_max_glob - t * SHARD_GRID_STEP
    return None


def decode_sharded(q: np.ndarray, shards: List[Index], p: float) -> dict:
    """Whole sequence-sharded decode for one unit (all shards in-process)."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    G = q.shape[0]
    S = len(shards)
    st1 = [[shard_stage1(q[g], shards[s]) for g in range(G)] for s in range(S)]
    m_glob = [max(st1[s][g]["m"] for s in range(S)) for g in range(G)]
    th_glob = [max(st1[s][g]["theta_max"] for s in range(S)) for g in range(G)]
    vecs = [[shard_mass_vector(st1[s][g], m_glob[g], th_glob[g]) for g in range(G)] for s in range(S)]
    tot = [sum(vecs[s][g] for s in range(S)) for g in range(G)]
    theta_star = [shard_threshold(tot[g], p, th_glob[g]) for g in range(G)]
    o_parts, lse_parts, unions = [], [], []
    for s in range(S):
        idx = shards[s]
        mask = np.zeros(idx.C, dtype=bool)
        for g in range(G):
            th = st1[s][g]["theta"]
            sel = (idx.sizes > 0) if theta_star[g] is None else ((th >= theta_star[g]) & (idx.sizes > 0))
            mask |= sel
        U = np.nonzero(mask)[0]
        unions.append(U)
        toks = cluster_tokens(idx, U)
        if toks.size == 0:
            o_parts.append(np.zeros((G, idx.K.shape[1])))
            lse_parts.append(np.full(G, -np.inf))
        else:
            o, lse = sparse_attention(q, idx.K, idx.V, toks)
            o_parts.append(o)
            lse_parts.append(lse)
    o, lse = lse_merge(np.array(o_parts), np.array(lse_parts))
    return {"o": o, "lse": lse, "unions": unions, "theta_star": theta_star,
            "m_glob": m_glob, "theta_max": th_glob, "mass_total": tot}
