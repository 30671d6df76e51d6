"""Pins for the CPU float64 oracle (runs without a GPU).

Every test checks the oracle against something other than itself: a library
routine (scikit-learn Lloyd, torch SDPA, scipy digamma), a closed form, brute
force on tiny inputs, an invariant the paper states, or a worked example copied
from SPEC.md into tests/golden/spec_examples.json.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
from scipy.special import digamma

from oracle import tactic_oracle as O
from synth import bf16_round, make_unit, uniform_unit

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_index(n, C, d=16, seed=0, iters=10):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((n, d))
    V = rng.standard_normal((n, d))
    idx, km = O.build_index(K, V, C, iters, seed=seed)
    return idx, km, rng


# ----------------------------------------------------------------------------- sampler
def test_init_sampler_properties():
    for n, C in [(10, 10), (4096, 64), (131072, 1024)]:
        a = O.init_indices(n, C, seed=3, unit=1)
        assert a.shape == (C,) and len(set(a.tolist())) == C
        assert a.min() >= 0 and a.max() < n
        assert np.array_equal(a, O.init_indices(n, C, seed=3, unit=1))
    assert not np.array_equal(O.init_indices(4096, 64, 0, 0), O.init_indices(4096, 64, 0, 1))
    # C = n draws a full permutation (partial Fisher-Yates run to the end)
    assert sorted(O.init_indices(50, 50, 1, 0).tolist()) == list(range(50))
    with pytest.raises(ValueError):
        O.init_indices(4, 5, 0, 0)


def test_init_sampler_uniform_marginals():
    # every token equally likely to be picked: chi-square over many seeds
    n, C, trials = 20, 5, 4000
    cnt = np.zeros(n)
    for s in range(trials):
        cnt[O.init_indices(n, C, s, 0)] += 1
    exp = trials * C / n
    chi2 = np.sum((cnt - exp) ** 2 / exp)
    assert chi2 < 45.0  # 19 dof, p ~ 1e-3


# ----------------------------------------------------------------------------- k-means
def test_kmeans_spec_examples():
    for ex in GOLD["kmeans"]:
        K = np.array(ex["keys"], dtype=float)
        km = O.kmeans(K, ex["C"], 10, init=ex.get("init", [0]))
        assert km["inertia"] == pytest.approx(ex["inertia"], abs=1e-12), ex["cite"]
        np.testing.assert_allclose(km["centroids"], np.array(ex["centroids"], dtype=float))
        if "members" in ex:
            idx = O.make_index(K, K, km["centroids"], km["assign"])
            mem = [sorted(idx.perm[idx.offsets[j]:idx.offsets[j + 1]].tolist()) for j in range(ex["C"])]
            assert mem == ex["members"]


def test_kmeans_matches_sklearn_lloyd():
    from sklearn.cluster import KMeans
    for seed in range(3):
        u = make_unit(1024, 1, seed=seed)
        K = u["K"].astype(np.float64)
        C = 8
        init = O.init_indices(1024, C, seed, 0)
        km = O.kmeans(K, C, 300, init=init)
        sk = KMeans(n_clusters=C, init=K[init], n_init=1, max_iter=300, tol=0.0,
                    algorithm="lloyd").fit(K)
        if np.min(km["sizes"]) == 0:
            continue  # sklearn relocates empty clusters; reading 6 keeps them
        assert np.array_equal(sk.labels_, km["assign"])
        np.testing.assert_allclose(sk.cluster_centers_, km["centroids"], rtol=1e-10, atol=1e-10)
        assert km["inertia"] == pytest.approx(sk.inertia_, rel=1e-9)


def test_kmeans_inertia_nonincreasing_and_invariants():
    u = make_unit(4096, 1, seed=1)
    K = u["K"].astype(np.float64)
    km = O.kmeans(K, 64, 10, seed=1)
    tr = km["inertia_trace"]
    assert all(tr[i + 1] <= tr[i] * (1 + 1e-12) for i in range(len(tr) - 1))
    a, c = km["assign"], km["centroids"]
    # centroids are exact member means (or untouched when empty)
    for j in range(64):
        m = a == j
        if m.any():
            np.testing.assert_allclose(c[j], K[m].mean(axis=0), rtol=1e-12, atol=1e-12)
    assert km["inertia"] == pytest.approx(float(np.sum((K - c[a]) ** 2)), rel=1e-12)


def test_kmeans_assignment_is_nearest_direct_distance():
    # brute-force squared distances written out per pair, not via the expansion
    rng = np.random.default_rng(5)
    K = rng.standard_normal((60, 6))
    c = rng.standard_normal((7, 6))
    a, _ = O._sq_dist_argmin(K, c)
    for i in range(60):
        dist = [sum((K[i, t] - c[j, t]) ** 2 for t in range(6)) for j in range(7)]
        assert a[i] == int(np.argmin(dist))
    # a tie resolves to the lowest id
    K2 = np.array([[0.0, 0.0]])
    c2 = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]])
    assert O._sq_dist_argmin(K2, c2)[0][0] == 0


def test_kmeans_discrete_partition_avg_size_one():
    rng = np.random.default_rng(2)
    K = rng.standard_normal((40, 5))
    km = O.kmeans(K, 40, 10, init=np.arange(40))
    assert km["inertia"] == 0.0
    assert sorted(km["assign"].tolist()) == list(range(40))


def test_kmeans_permutation_invariance():
    rng = np.random.default_rng(9)
    K = np.concatenate([rng.standard_normal((50, 4)) + 8 * k for k in range(4)])
    init = np.array([0, 50, 100, 150])
    km1 = O.kmeans(K, 4, 20, init=init)
    pi = rng.permutation(200)
    inv = np.argsort(pi)
    km2 = O.kmeans(K[pi], 4, 20, init=inv[init])
    part1 = {frozenset(np.nonzero(km1["assign"] == j)[0]) for j in range(4)}
    part2 = {frozenset(pi[np.nonzero(km2["assign"] == j)[0]]) for j in range(4)}
    assert part1 == part2


def test_layout_partition_and_order():
    idx, km, _ = _rand_index(500, 12)
    perm, off = idx.perm, idx.offsets
    assert sorted(perm.tolist()) == list(range(500))
    for j in range(12):
        seg = perm[off[j]:off[j + 1]]
        assert np.all(km["assign"][seg] == j)
        assert np.all(np.diff(seg) > 0)


# ----------------------------------------------------------------------------- ranking
def test_ranking_spec_example():
    ex = GOLD["ranking"][0]
    c = np.array(ex["centroids"])
    idx = O.make_index(c, c, c, np.arange(2))
    crit = O.criticality(np.array(ex["q"]), idx)
    assert O.sort_clusters(crit).tolist() == ex["order"], ex["cite"]


def test_ranking_singleton_clusters_equals_true_score_order():
    # C = n: every key is its own centroid, so pi must be the exact attention order
    rng = np.random.default_rng(3)
    K = bf16_round(rng.standard_normal((64, 8)).astype(np.float32)).astype(np.float64)
    q = rng.standard_normal(8)
    idx = O.make_index(K, K, K, np.arange(64))
    order = O.sort_clusters(O.criticality(q, idx))
    s = O.exact_scores(q, K)
    assert np.all(np.diff(s[order]) <= 0)
    assert np.array_equal(order, np.argsort(-s, kind="stable"))


def test_ranking_scale_invariance_and_ties():
    idx, _, rng = _rand_index(300, 10)
    q = rng.standard_normal(16)
    o1 = O.sort_clusters(O.criticality(q, idx))
    o2 = O.sort_clusters(O.criticality(3.5 * q, idx))
    assert np.array_equal(o1, o2)
    assert O.sort_clusters(np.array([1.0, 2.0, 2.0, 0.0])).tolist() == [1, 2, 0, 3]


# ----------------------------------------------------------------------------- fitting / budget
def test_fit_two_point_defining_property():
    rng = np.random.default_rng(0)
    for _ in range(100):
        x1, x2 = sorted(rng.integers(1, 10000, size=2) + np.array([0, 1]))
        mu1, mu2 = rng.random(2)
        a, b = O.fit_two_point(float(x1), mu1, float(x2), mu2)
        assert a / x1 + b == pytest.approx(mu1, rel=1e-12, abs=1e-14)
        assert a / x2 + b == pytest.approx(mu2, rel=1e-12, abs=1e-14)


def test_fit_noiseless_and_constant():
    a0, b0 = 3.7, 0.02
    a, b = O.fit_two_point(10.0, a0 / 10 + b0, 60.0, a0 / 60 + b0)
    assert a == pytest.approx(a0, rel=1e-9) and b == pytest.approx(b0, rel=1e-9)
    a, b = O.fit_two_point(10.0, 0.4, 60.0, 0.4)
    assert a == 0.0 and b == pytest.approx(0.4)


def test_token_budget_spec_examples():
    for ex in GOLD["budget"]:
        n = ex["n"]
        w = 1.0 / np.arange(1, n + 1) if ex["weights"] == "harmonic" else np.ones(n)
        assert O.token_budget(w, ex["P"]) == ex["k"], ex["cite"]


def test_token_budget_shift_invariance():
    rng = np.random.default_rng(4)
    w = rng.random(200)
    for P in [0.3, 0.7, 0.95]:
        assert O.token_budget(w, P) == O.token_budget(w * 1e-30, P) == O.token_budget(w * 7e20, P)


def _harmonic(k):
    return digamma(np.asarray(k, dtype=float) + 1.0) + np.euler_gamma


def test_estimated_mass_matches_clamp_aware_harmonic_closed_form():
    for seed in range(4):
        u = make_unit(4096, 2, seed=seed)
        idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=seed)
        for g in range(2):
            h = O.decode_head(u["q"][g], idx, 0.9)
            n, N, a, b = idx.n, h["N"], h["a"], h["b"]
            E_N = float(np.sum(h["what"][:N]))
            for e in [N + 1, N + 7, 1000, 2048, n]:
                i = np.arange(N + 1, e + 1, dtype=float)
                if a >= 0 and b >= 0:
                    F = a * (_harmonic(e) - _harmonic(N)) + b * (e - N)
                elif a > 0 > b:
                    top = min(e, int(np.floor(a / -b)))
                    while top > N and a / top + b <= 0:
                        top -= 1
                    F = a * (_harmonic(top) - _harmonic(N)) + b * (top - N) if top > N else 0.0
                elif a <= 0 and b <= 0:
                    F = 0.0
                else:
                    lo = max(N + 1, int(np.floor(-a / b)) + 1)
                    while lo <= e and a / lo + b <= 0:
                        lo += 1
                    F = a * (_harmonic(e) - _harmonic(lo - 1)) + b * (e - lo + 1) if lo <= e else 0.0
                cum = float(np.sum(h["what"][:e]))
                assert cum == pytest.approx(E_N + F, rel=1e-10)


def test_sample_constants_follow_paper_fractions():
    for n in [4096, 32768, 131072, 1048576]:
        sc = O.sample_constants(n)
        assert 0.02 * n <= sc["N"] < 0.02 * n + 1           # P:376 "1-2%" (upper end)
        assert abs(sc["x1"] - 0.1 * n) <= 0.5                # P:373 "10%"
        assert abs(sc["x2"] - 0.6 * n) <= 0.5                # P:373 "60%"
        assert abs(sc["w"] - 0.0025 * n) <= 0.5 or sc["w"] == 1
        assert not sc["fallback"]
    assert O.sample_constants(10)["fallback"]


def test_sample_constants_ppm_rule_defaults_are_the_integer_formulas():
    """Readings 8-10: with the default fractions the ppm rule reproduces the integer
    formulas N = (2n+99) div 100, x1 = (n+5) div 10, x2 = (6n+5) div 10,
    w = max(1, (25n+5000) div 10000) for every n (checked exhaustively to 2^17 and on
    a sample up to 2^20), whether the fractions arrive as float64 or float32."""
    ns = list(range(1, 1 << 17)) + list(np.random.default_rng(0).integers(1 << 17, (1 << 20) + 1, 3000))
    for f32 in (False, True):
        conv = (lambda v: float(np.float32(v))) if f32 else float
        kw = {k: conv(v) for k, v in O.DEFAULT_SAMPLING.items()}
        for n in ns[:: (1 if not f32 else 7)]:
            n = int(n)
            sc = O.sample_constants(n, **kw)
            assert (sc["N"], sc["x1"], sc["x2"], sc["w"]) == (
                (2 * n + 99) // 100, (n + 5) // 10, (6 * n + 5) // 10, max(1, (25 * n + 5000) // 10000)), n


def test_sample_constants_custom_fractions():
    # P:376 "1-2%": the lower end; windows at 20% / 50% with a 1% half-width
    sc = O.sample_constants(100000, exact_frac=0.01, p1=0.2, p2=0.5, window_half_frac=0.01)
    assert (sc["N"], sc["x1"], sc["x2"], sc["w"], sc["fallback"]) == (1000, 20000, 50000, 1000, False)
    sc = O.sample_constants(999, exact_frac=0.015, p1=0.25, p2=0.75, window_half_frac=0.001)
    assert (sc["N"], sc["x1"], sc["x2"], sc["w"]) == (15, 250, 749, 1)   # 14.985 up, 249.75, 749.25, 0.999
    for bad in [dict(p1=0.6, p2=0.1), dict(exact_frac=0.0), dict(window_half_frac=0.0), dict(p2=1.0)]:
        with pytest.raises(ValueError):
            O.sample_constants(1000, **bad)


def test_splitmix64_known_answer_vector():
    """The init sampler's generator is SplitMix64 (reading 3): its published first outputs
    from state 0 (Steele, Lea & Flood's reference stream)."""
    g = O._splitmix64_stream(0)
    assert [next(g) for _ in range(5)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
                                           0xF88BB8A8724C81EC, 0x1B39896A51A8749B]


def _planted_harmonic_unit(n, a_star, b_star, seed=0, d=128):
    """Singleton clusters whose exact weight at sorted rank i is proportional to
    a*/i + b*: key i has component 0 = log(a*/r_i + b*) for a random rank r_i (the
    other components random), the query points along component 0 with |q| = sqrt(d),
    so the logit q.k/sqrt(d) is that log up to rounding."""
    rng = np.random.default_rng(seed)
    ranks = rng.permutation(n) + 1                    # token i has rank ranks[i]
    K = rng.standard_normal((n, d)) * 0.3
    K[:, 0] = np.log(a_star / ranks + b_star)
    V = rng.standard_normal((n, d))
    q = np.zeros(d)
    q[0] = np.sqrt(d)
    idx = O.make_index(K, V, K, np.arange(n))         # C = n, centroid = key
    return idx, q, ranks


@pytest.mark.parametrize("n,a_star,b_star", [(2000, 3.0, 0.01), (2000, 0.5, 0.0), (12345, 7.0, 0.002)])
def test_window_means_and_fit_on_planted_harmonic_weights(n, a_star, b_star):
    """O7 pinned independently (Alg. 1 l.4): on an
    instance whose exp-logit at sorted rank i is exactly proportional to a*/i + b*, the
    shift m is the rank-1 logit, the exact head is (a*/i + b*)/y_1 for i <= N, and each
    window mean is the harmonic closed form
        mu_k = (a* (H(x_k + w) - H(x_k - w - 1)) / (2w + 1) + b*) / y_1,
    with H from scipy's digamma; the fitted a/x + b passes through (x_k, mu_k).  A
    sum instead of a mean, a window shifted by one rank, or a wrong shift fails it."""
    idx, q, ranks = _planted_harmonic_unit(n, a_star, b_star)
    h = O.decode_head(q, idx, 0.9)
    N, x1, x2, w = h["N"], h["x1"], h["x2"], h["w"]
    assert not h["fallback"]
    y1 = a_star + b_star
    # the order is descending weight: rank r holds the token with ranks[token] == r
    tok = np.argsort(ranks)
    assert np.array_equal(h["order"], tok)
    assert h["m"] == pytest.approx(np.log(y1), abs=1e-12)
    i = np.arange(1, N + 1)
    np.testing.assert_allclose(h["what"][:N], (a_star / i + b_star) / y1, rtol=1e-12)
    for x, mu in ((x1, h["mu1"]), (x2, h["mu2"])):
        expect = (a_star * (_harmonic(x + w) - _harmonic(x - w - 1)) / (2 * w + 1) + b_star) / y1
        assert mu == pytest.approx(expect, rel=1e-12)
    for x, mu in ((x1, h["mu1"]), (x2, h["mu2"])):
        assert h["a"] / x + h["b"] == pytest.approx(mu, rel=1e-12)
    # and the fitted curve's tail beyond N is clamp-free: W = E_N + a (H(n) - H(N)) + b (n - N)
    if h["a"] >= 0 and h["b"] >= 0:
        W = float(np.sum(h["what"][:N])) + h["a"] * (_harmonic(n) - _harmonic(N)) + h["b"] * (n - N)
        assert h["W"] == pytest.approx(W, rel=1e-10)


def test_window_means_with_custom_sampling_fractions():
    """Same planted instance through non-default fractions (P:376 lower end 1%, windows at
    20% / 50% with a 0.5% half-width): the means follow the constants of the ppm rule."""
    n, a_star, b_star = 5000, 2.0, 0.004
    idx, q, _ = _planted_harmonic_unit(n, a_star, b_star, seed=3)
    smp = dict(exact_frac=0.01, p1=0.2, p2=0.5, window_half_frac=0.005)
    h = O.decode_head(q, idx, 0.9, sampling=smp)
    assert (h["N"], h["x1"], h["x2"], h["w"]) == (50, 1000, 2500, 25)
    y1 = a_star + b_star
    for x, mu in ((h["x1"], h["mu1"]), (h["x2"], h["mu2"])):
        expect = (a_star * (_harmonic(x + 25) - _harmonic(x - 26)) / 51 + b_star) / y1
        assert mu == pytest.approx(expect, rel=1e-12)


# ----------------------------------------------------------------------------- selection
def test_selection_monotone_in_p_and_p1_selects_all():
    u = make_unit(4096, 4, seed=2)
    idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=2)
    for g in range(4):
        prev = set()
        for p in [0.3, 0.5, 0.8, 0.9, 0.95, 0.99, 1.0]:
            S = set(O.decode_head(u["q"][g], idx, p)["S"].tolist())
            assert prev <= S
            prev = S
        assert prev == set(np.nonzero(idx.sizes > 0)[0].tolist())


def test_selection_equals_token_budget_rounded_to_cluster_end():
    # O10 at cluster granularity == Alg. 1's k* rounded up to the end of its cluster
    u = make_unit(4096, 4, seed=5)
    idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=5)
    for g in range(4):
        for p in [0.5, 0.9]:
            h = O.decode_head(u["q"][g], idx, p)
            k = O.token_budget(h["what"], p)
            J = int(np.searchsorted(h["ends"], k)) + 1    # first cluster whose end >= k
            assert J == h["J"]


def test_logit_shift_invariance():
    u = make_unit(4096, 1, seed=6)
    K = u["K"].astype(np.float64)
    q = u["q"][0].astype(np.float64)
    km = O.kmeans(K, 64, 10, seed=6)
    shift = 3.0 * np.sqrt(K.shape[1]) * q / (q @ q)       # adds +3 to every logit
    i1 = O.make_index(K, u["V"], km["centroids"], km["assign"])
    i2 = O.Index(K + shift, i1.V, i1.assign, i1.centroids + shift, i1.offsets, i1.perm, i1.sizes, i1.C)
    h1, h2 = O.decode_head(q, i1, 0.9), O.decode_head(q, i2, 0.9)
    assert np.array_equal(h1["order"], h2["order"]) and h1["J"] == h2["J"]
    assert h2["m"] == pytest.approx(h1["m"] + 3.0, rel=1e-9)
    assert h2["a"] == pytest.approx(h1["a"], rel=1e-7) and h2["b"] == pytest.approx(h1["b"], rel=1e-6, abs=1e-12)


def test_optimal_budget_is_brute_force_minimum():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(3, 11))
        K = rng.standard_normal((n, 4)) * 2
        q = rng.standard_normal(4)
        s = O.exact_scores(q, K)
        for P in [0.3, 0.6, 0.9]:
            best = None
            for k in range(1, n + 1):
                if any(s[list(c)].sum() >= P for c in itertools.combinations(range(n), k)):
                    best = k
                    break
            assert O.optimal_budget(q, K, P) == best


def test_fallback_tiny_n_is_cluster_optimal():
    rng = np.random.default_rng(12)
    for trial in range(10):
        n, C = 12, 4
        K = rng.standard_normal((n, 8)) * 1.5
        V = rng.standard_normal((n, 8))
        q = rng.standard_normal(8)
        idx, _ = O.build_index(K, V, C, 10, seed=trial)
        assert O.sample_constants(n)["fallback"]
        for P in [0.5, 0.9]:
            h = O.decode_head(q, idx, P)
            assert int(idx.sizes[h["S"]].sum()) == O.cluster_optimal_budget(q, idx, P)


def test_union_superset_and_table1_ordering():
    u = make_unit(4096, 4, seed=7)
    idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=7)
    r = O.decode_unit(u["q"], idx, 0.9)
    for g, h in enumerate(r["heads"]):
        assert set(h["S"].tolist()) <= set(r["U"].tolist())
        pU = O.cumulative_score(u["q"][g], idx.K, r["tokens"])
        pS = O.cumulative_score(u["q"][g], idx.K, O.cluster_tokens(idx, h["S"]))
        assert pU >= pS - 1e-15
        # Table 1 column order: Optimal <= Cluster-Optimal
        assert O.optimal_budget(u["q"][g], idx.K, 0.9) <= O.cluster_optimal_budget(u["q"][g], idx, 0.9)


def test_table1_success_semantics():
    ex = GOLD["table1_semantics"][0]
    assert (ex["achieved"] >= ex["threshold"]) == ex["success"]
    for row in GOLD["table1_paper"]:
        assert row["optimal"] <= row["cluster_optimal"] <= row["tactic"], row["cite"]


# ----------------------------------------------------------------------------- attention
def _sdpa(q, K, V):
    qt = torch.tensor(np.atleast_2d(q), dtype=torch.float64)[None]
    Kt = torch.tensor(K, dtype=torch.float64)[None]
    Vt = torch.tensor(V, dtype=torch.float64)[None]
    return torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt)[0].numpy()


def test_full_attention_matches_torch_sdpa():
    rng = np.random.default_rng(1)
    q, K, V = rng.standard_normal((4, 128)), rng.standard_normal((300, 128)) * 3, rng.standard_normal((300, 128))
    o, lse = O.full_attention(q, K, V)
    np.testing.assert_allclose(o, _sdpa(q, K, V), rtol=1e-12, atol=1e-12)
    from scipy.special import logsumexp
    np.testing.assert_allclose(lse, logsumexp(q @ K.T / np.sqrt(128), axis=1), rtol=1e-13)


def test_p1_decode_equals_full_attention():
    u = make_unit(4096, 4, seed=3)
    idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=3)
    r = O.decode_unit(u["q"], idx, 1.0)
    np.testing.assert_allclose(r["o"], _sdpa(u["q"].astype(float), u["K"].astype(float), u["V"].astype(float)),
                               rtol=1e-11, atol=1e-12)


def test_attention_special_cases():
    rng = np.random.default_rng(8)
    K, V, q = rng.standard_normal((50, 16)), rng.standard_normal((50, 16)), rng.standard_normal(16)
    o, _ = O.sparse_attention(q, K, V, [17])                     # S:347 single token -> v_j
    np.testing.assert_allclose(o[0], V[17], rtol=1e-15)
    Vc = np.tile(rng.standard_normal(16), (50, 1))                # S:337 constant V -> V
    np.testing.assert_allclose(O.full_attention(q, K, Vc)[0][0], Vc[0], rtol=1e-13)
    assert O.exact_scores(q, K).sum() == pytest.approx(1.0, rel=1e-14)   # softmax mass = 1
    with pytest.raises(ValueError):
        O.sparse_attention(q, K, V, [])


def test_lse_merge_split_anywhere_and_associative():
    rng = np.random.default_rng(2)
    q, K, V = rng.standard_normal((3, 32)), rng.standard_normal((200, 32)) * 2, rng.standard_normal((200, 32))
    o_full, lse_full = O.full_attention(q, K, V)
    cuts = [0, 13, 14, 90, 200]
    parts = [O.full_attention(q, K[a:b], V[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    o, lse = O.lse_merge(np.array([p[0] for p in parts]), np.array([p[1] for p in parts]))
    np.testing.assert_allclose(o, o_full, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(lse, lse_full, rtol=1e-13)
    # ((A+B)+C) == (A+(B+C)) == permuted
    A, B, Cc = parts[0], parts[1], parts[2]
    ab = O.lse_merge(np.array([A[0], B[0]]), np.array([A[1], B[1]]))
    bc = O.lse_merge(np.array([B[0], Cc[0]]), np.array([B[1], Cc[1]]))
    l1 = O.lse_merge(np.array([ab[0], Cc[0]]), np.array([ab[1], Cc[1]]))
    l2 = O.lse_merge(np.array([A[0], bc[0]]), np.array([A[1], bc[1]]))
    l3 = O.lse_merge(np.array([Cc[0], A[0], B[0]]), np.array([Cc[1], A[1], B[1]]))
    for x in (l2, l3):
        np.testing.assert_allclose(x[0], l1[0], rtol=1e-12, atol=1e-14)


def test_appendix_a_bound_random_and_selected():
    rng = np.random.default_rng(0)
    for _ in range(1000):                                       # S:357 / S:560
        n = int(rng.integers(2, 40))
        K, V, q = rng.standard_normal((n, 8)) * 2, rng.standard_normal((n, 8)), rng.standard_normal(8)
        I = rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False)
        assert O.attention_distance(q, K, V, I) <= O.distance_bound(q, K, V, I) + 1e-12
    u = make_unit(4096, 4, seed=4)
    idx, _ = O.build_index(u["K"], u["V"], 64, 10, seed=4)
    r = O.decode_unit(u["q"], idx, 0.9)
    for g in range(4):
        eps = np.linalg.norm(O.full_attention(u["q"][g], idx.K, idx.V)[0][0] - r["o"][g])
        assert eps <= O.distance_bound(u["q"][g], idx.K, idx.V, r["tokens"]) + 1e-12


def test_kl_example():
    ex = GOLD["kl"][0]
    p, q = np.array(ex["p"]), np.array(ex["q"])
    m = p > 0
    assert float(np.sum(p[m] * np.log(p[m] / q[m]))) == pytest.approx(np.log(2.0))


# ----------------------------------------------------------------------------- sharded rule
def test_sharded_p1_equals_full_attention_and_covers_single_rule():
    u = make_unit(8192, 4, seed=1)
    K, V, q = u["K"], u["V"], u["q"]
    S = 4
    shards = []
    for s in range(S):
        sl = slice(s * 2048, (s + 1) * 2048)
        shards.append(O.build_index(K[sl], V[sl], 32, 10, seed=1, unit=s)[0])
    r1 = O.decode_sharded(q, shards, 1.0)
    np.testing.assert_allclose(r1["o"], _sdpa(q.astype(float), K.astype(float), V.astype(float)), rtol=1e-10, atol=1e-12)
    r = O.decode_sharded(q, shards, 0.9)
    # the global rule reaches its threshold on the estimated mass; p(U) of the exact
    # scores is reported (not asserted) like Table 1.  Structural checks only:
    for g in range(4):
        assert r["theta_star"][g] is None or r["theta_star"][g] <= r["theta_max"][g]
        tot = r["mass_total"][g]
        assert np.all(np.diff(tot[1:]) >= -1e-12 * tot[0])    # M(theta) monotone in the grid
    # S = 1 shard: the grid rule is conservative -> superset of the exact-threshold union
    full = O.build_index(K, V, 64, 10, seed=1)[0]
    rs = O.decode_sharded(q, [full], 0.9)
    ru = O.decode_unit(q, full, 0.9)
    assert set(ru["U"].tolist()) <= set(rs["unions"][0].tolist())


# ----------------------------------------------------------------------------- generator
def test_generator_deterministic_bf16_exact():
    a = make_unit(2048, 4, seed=9, b=1, h=2)
    b = make_unit(2048, 4, seed=9, b=1, h=2)
    for k in ("K", "V", "q"):
        assert np.array_equal(a[k], b[k])
        assert np.array_equal(bf16_round(a[k]), a[k])
    assert a["K"].shape == (2048, 128) and a["q"].shape == (4, 128)
    c = make_unit(2048, 4, seed=9, b=1, h=3)
    assert not np.array_equal(a["K"], c["K"])
    vn = np.linalg.norm(a["V"], axis=1)
    assert 0.7 < vn.min() and vn.max() < 1.3                  # near-constant |v| (Fig. 2)
    uu = uniform_unit(100, 2, 0)
    assert uu["K"].shape == (100, 128)


# ----------------------------------------------------------------------------- NEXT 1: multi-step generation
def test_assign_tokens_is_brute_force_nearest_with_lowest_id_ties():
    """SPEC assign_token: nearest centroid by direct squared distances,
    ties to the lowest id -- pinned by a per-pair loop and deliberate duplicate centroids."""
    rng = np.random.default_rng(11)
    c = rng.standard_normal((9, 8))
    c[5] = c[2]                      # exact duplicate: ties must go to id 2
    k = np.concatenate([rng.standard_normal((40, 8)), c[[2, 7]] + 0.0])
    got = O.assign_tokens(k, c)
    for i, ki in enumerate(k):
        d = [float(((ki - cj) ** 2).sum()) for cj in c]
        best = min(d)
        assert got[i] == d.index(best)
    assert got[-2] == 2 and got[-1] == 7


def test_tail_decode_p1_equals_full_attention_over_all_tokens():
    """p = 1 selects every cluster (reading 15), so decode with a tail of appended tokens
    equals full attention over the n + t tokens (torch SDPA, independent of the oracle)."""
    u = make_unit(2048, 4, seed=5)
    idx, _ = O.build_index(u["K"], u["V"], 32, 3, seed=5)
    rng = np.random.default_rng(5)
    Kt = bf16_round(rng.standard_normal((19, 128)).astype(np.float32))
    Vt = bf16_round(rng.standard_normal((19, 128)).astype(np.float32))
    r = O.decode_unit_with_tail(u["q"], idx, 1.0, Kt, Vt)
    K_all = torch.from_numpy(np.concatenate([u["K"], Kt]).astype(np.float64))
    V_all = torch.from_numpy(np.concatenate([u["V"], Vt]).astype(np.float64))
    q = torch.from_numpy(u["q"].astype(np.float64))
    ref = torch.nn.functional.scaled_dot_product_attention(q[None, :, None, :], K_all[None, None].expand(1, 4, -1, -1),
                                                           V_all[None, None].expand(1, 4, -1, -1))[0, :, 0]
    np.testing.assert_allclose(r["o"], ref.numpy(), atol=1e-12, rtol=1e-10)


def test_tail_decode_is_lse_merge_of_union_and_tail_and_empty_tail_is_plain_decode():
    """The tail adds one more LSE-mergeable part: attention over U + tail equals the
    merge of attention over U and attention over the tail; an empty tail changes nothing."""
    u = make_unit(4096, 4, seed=6)
    idx, _ = O.build_index(u["K"], u["V"], 64, 3, seed=6)
    rng = np.random.default_rng(6)
    Kt = bf16_round(rng.standard_normal((33, 128)).astype(np.float32))
    Vt = bf16_round(rng.standard_normal((33, 128)).astype(np.float32))
    base = O.decode_unit(u["q"], idx, 0.9)
    r = O.decode_unit_with_tail(u["q"], idx, 0.9, Kt, Vt)
    assert np.array_equal(r["union_mask"], base["union_mask"])   # the selection ignores the tail
    ot, lt = O.full_attention(u["q"], Kt, Vt)
    om, lm = O.lse_merge(np.stack([base["o"], ot]), np.stack([base["lse"], lt]))
    np.testing.assert_allclose(r["o"], om, atol=1e-12)
    np.testing.assert_allclose(r["lse"], lm, atol=1e-12)
    r0 = O.decode_unit_with_tail(u["q"], idx, 0.9, np.zeros((0, 128)), np.zeros((0, 128)))
    np.testing.assert_allclose(r0["o"], base["o"], atol=0)


# ----------------------------------------------------------------------------- NEXT 4: fixed-budget baseline
def test_fixed_budget_singletons_is_top_k_true_scores_and_rounds_to_cluster_end():
    """SPEC fixed_budget_select: with singleton clusters the criticality order is
    the true score order, so a budget of k tokens is the top-k tokens; with real clusters
    the set closes at the first cluster end reaching k."""
    rng = np.random.default_rng(8)
    n = 64
    K = bf16_round(rng.standard_normal((n, 16)).astype(np.float32))
    V = bf16_round(rng.standard_normal((n, 16)).astype(np.float32))
    idx = O.make_index(K, V, K.astype(np.float64), np.arange(n))
    q = bf16_round(rng.standard_normal(16).astype(np.float32))
    for k in (1, 7, 33, 64):
        r = O.fixed_budget_select(q, idx, k)
        top = np.argsort(-(K.astype(np.float64) @ q.astype(np.float64)), kind="stable")[:k]
        assert sorted(O.cluster_tokens(idx, r["S"]).tolist()) == sorted(top.tolist())
    idx2, _, _ = _rand_index(256, 16, seed=8)
    q2 = rng.standard_normal(16)
    for k in (1, 50, 200, 256):
        r = O.fixed_budget_select(q2, idx2, k)
        ends = np.cumsum(idx2.sizes[r["order"]])
        assert ends[r["J"] - 1] >= k and (r["J"] == 1 or ends[r["J"] - 2] < k)


def test_windows_exact_variant_weights_and_total():
    """SPEC S:284 / S:297 variant: window ranks carry their exact weights; the estimated
    total changes by exactly sum(exact - fitted) over the window ranks, the rest of the
    weights are unchanged, and the selection stays monotone in p."""
    u = make_unit(8192, 4, seed=9)
    idx, _ = O.build_index(u["K"], u["V"], 128, 3, seed=9)
    q = u["q"][0]
    a = O.decode_head(q, idx, 0.9)
    b = O.decode_head(q, idx, 0.9, windows_exact=True)
    sc = O.sample_constants(idx.n)
    win = np.concatenate([np.arange(sc["x1"] - sc["w"], sc["x1"] + sc["w"] + 1),
                          np.arange(sc["x2"] - sc["w"], sc["x2"] + sc["w"] + 1)]) - 1
    tok = O.sorted_tokens(idx, b["order"])
    ell = (idx.K[tok[win]] @ q.astype(np.float64)) / np.sqrt(128)
    np.testing.assert_allclose(b["what"][win], np.exp(ell - b["m"]), rtol=1e-12)
    rest = np.ones(idx.n, dtype=bool)
    rest[win] = False
    np.testing.assert_array_equal(a["what"][rest], b["what"][rest])
    assert b["W"] - a["W"] == pytest.approx(float(b["what"][win].sum() - a["what"][win].sum()), rel=1e-9, abs=1e-12)
    Js = [O.decode_head(q, idx, p, windows_exact=True)["J"] for p in (0.5, 0.8, 0.9, 0.95, 0.99)]
    assert Js == sorted(Js)


# ---------------------------------------------------------------------------- frozen input recipe
def test_recipe_regression_pins():
    """The frozen recipe (tactic-synth-v1) and the oracle's selection on it:
    per-head selected clusters and tokens and the GQA union at C1 and one 32K unit must stay
    exactly those recorded in tests/golden/recipe_regression.json (written by
    tools/make_recipe_golden.py, which calls only oracle/ and synth/) -- a change to the
    generator or to the oracle's arithmetic shows up here first."""
    import json
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import make_recipe_golden as M
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "recipe_regression.json")))
    assert gold["recipe"] == "tactic-synth-v1"
    for g in gold["cases"]:
        got = M.compute(g["case"])
        assert got["inertia"] == pytest.approx(g["inertia"], rel=1e-12)
        assert got["p"] == g["p"], g["case"]["name"]
