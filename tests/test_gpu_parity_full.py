"""GPU parity at the headline sizes (BASELINE.json configs[1], C2: 8 units x 131072 tokens,
C = 1024) and at the other configurations the bench times, against the float64 oracle:

* the tcgen05 k-means (B1-B4) from an identical init at C = 1024 (8 centroid
  tiles, the barrier phase wraps) and C = 4096: inertia within 1e-4 relative;
* the decode on the index the GPU itself built -- exactly what bench.py times -- against
  the oracle's decode on that clustering (exported), for every unit: order exact, J within
  the threshold band, union = the oracle order's prefixes, output within 2e-2 / 5e-3;
* the dense split-KV baseline (S10) at 131072 tokens against full attention;
* non-default Alg. 1 sampling fractions through the C ABI.
"""
import numpy as np
import pytest
import torch

from oracle import tactic_oracle as O
from synth import make_layer
from tests._gpu_helpers import (assert_output_close, assert_same_decode, dev_bf16, j_mismatch_allowed,
                                oracle_layer_clustering)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    from paper_2502_12216_b200 import build as B
    B.build()
    from paper_2502_12216_b200 import tactic
    tactic.device_check()
    return tactic


@pytest.fixture(scope="module")
def c2_layer():
    return make_layer(1, 8, 4, 131072, seed=0)


def _check_selection(res, u, G, heads_o, p, idx):
    for g in range(G):
        ho = heads_o[g]
        assert np.array_equal(res["order"][u, g], ho["order"]), f"order u{u} g{g}"
        assert j_mismatch_allowed(ho, int(res["J"][u, g]), p), f"J u{u} g{g}: {res['J'][u, g]} vs {ho['J']}"
        fit = res["fit"][u, g]
        if not ho["fallback"]:
            assert fit[2] == pytest.approx(ho["m"], abs=2e-5)
            assert fit[4] == pytest.approx(ho["mu1"], rel=2e-5)
            assert fit[5] == pytest.approx(ho["mu2"], rel=2e-5)
        assert fit[3] == pytest.approx(ho["W"], rel=1e-5)
    mask = np.zeros(idx.C, dtype=bool)
    for g in range(G):
        pos = heads_o[g]["order"][:res["J"][u, g]]
        mask[pos[idx.sizes[pos] > 0]] = True
    assert np.array_equal(mask, res["union_mask"][u]), f"union u{u}"


# ----------------------------------------------------------------------------- B2 at the headline cluster counts
@pytest.mark.slow
@pytest.mark.parametrize("C,iters", [(1024, 10), (4096, 4)])
def test_gpu_kmeans_inertia_parity_at_headline_cluster_counts(T, c2_layer, C, iters):
    """P:364 (§4.2) k-means, identical init on both sides: C = 1024 streams 8 centroid tiles
    per CTA (the mbarrier phase wraps), C = 4096 streams 32."""
    K, V, _ = c2_layer
    n = K.shape[2]
    units = 1
    init = np.stack([O.init_indices(n, C, 17, u) for u in range(units)]).astype(np.int32)
    Ku, Vu = K[:, :units], V[:, :units]
    index = T.build_index(dev_bf16(Ku), dev_bf16(Vu), C, iters, group_size=4, init=init)
    ex = index.export()
    for u in range(units):
        km = O.kmeans(Ku[0, u], C, iters, init=init[u])
        assert ex["inertia"][u] == pytest.approx(km["inertia"], rel=1e-4), (C, u)
        assert np.mean(ex["assign"][u] == km["assign"]) > 0.99
        assert ex["iters_run"][u] == km["iters_run"] or abs(ex["inertia"][u] - km["inertia"]) <= 1e-5 * km["inertia"]


# ----------------------------------------------------------------------------- the benchmarked path itself
@pytest.mark.slow
def test_gpu_built_c2_index_decode_matches_oracle_on_that_clustering(T, c2_layer):
    """bench.py's exact configuration: the C2 layer, index built on the GPU (tcgen05 k-means,
    10 iterations), decode at p = 0.9 and 0.5 -- every unit against the oracle's decode
    on the GPU's own exported clustering."""
    K, V, q = c2_layer
    G, C = 4, 1024
    index = T.build_index(dev_bf16(K), dev_bf16(V), C, 10, group_size=G, seed=0)
    ex = index.export()
    idxs = [O.make_index(K[0, u], V[0, u], ex["centroids"][u], ex["assign"][u]) for u in range(8)]
    qd = dev_bf16(q)
    for p in (0.9, 0.5):
        res = T.decode_debug(qd, index, p)
        got = res["out"].float().cpu().numpy()
        for u in range(8):
            qo = q[0, u * G:(u + 1) * G]
            ro = O.decode_unit(qo, idxs[u], p)
            _check_selection(res, u, G, ro["heads"], p, idxs[u])
            toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
            o, lse = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
            assert_output_close(got[0, u * G:(u + 1) * G], o, f"GPU-built C2 p={p} u={u}")
            np.testing.assert_allclose(res["lse"][0, u * G:(u + 1) * G].cpu().numpy(), lse, atol=2e-3)


@pytest.mark.slow
def test_dense_decode_at_131072_tokens(T, c2_layer):
    """S10, the library's own baseline, on the C2 layer (8 units x 131072 tokens) against
    full attention (Eq. 1-2)."""
    K, V, q = c2_layer
    G = 4
    lse = torch.empty((1, 32), dtype=torch.float32, device="cuda")
    out = T.dense_decode(dev_bf16(q), dev_bf16(K), dev_bf16(V), lse=lse).float().cpu().numpy()
    for u in range(8):
        o, l = O.full_attention(q[0, u * G:(u + 1) * G], K[0, u], V[0, u])
        assert_output_close(out[0, u * G:(u + 1) * G], o, f"dense 128K u={u}")
        np.testing.assert_allclose(lse[0, u * G:(u + 1) * G].cpu().numpy(), l, atol=2e-3)


# ----------------------------------------------------------------------------- sampling fractions through the ABI
@pytest.mark.parametrize("smp", [dict(exact_frac=0.01, p1=0.2, p2=0.5, window_half_frac=0.005),
                                 dict(exact_frac=0.015, p1=0.05, p2=0.7, window_half_frac=0.001)])
def test_custom_sampling_fractions_match_oracle(T, smp):
    """tactic_params_t's Alg. 1 fractions (P:373 window centres, P:376 exact share,
    reading 8 half-width): the index derives the oracle's constants and decodes like it."""
    G, n, C = 4, 32768, 256
    K, V, q = make_layer(1, 2, G, n, seed=44)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 44)
    index = T.import_index(dev_bf16(K), dev_bf16(V), cents, asg, group_size=G, sampling=smp)
    sc = index.sample_constants()
    ref = O.sample_constants(n, **smp)
    assert {k: sc[k] for k in ref} == ref
    qd = dev_bf16(q)
    for p in (0.8, 0.9):
        res = T.decode_debug(qd, index, p)
        got = res["out"].float().cpu().numpy()
        for u in range(2):
            qo = q[0, u * G:(u + 1) * G]
            ro = O.decode_unit(qo, idxs[u], p, sampling=smp)
            _check_selection(res, u, G, ro["heads"], p, idxs[u])
            toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
            o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
            assert_output_close(got[0, u * G:(u + 1) * G], o, f"sampling {smp} p={p} u={u}")


def test_bad_sampling_fractions_rejected(T):
    K, V, q = make_layer(1, 1, 4, 1024, seed=2)
    for bad in [dict(p1=0.7, p2=0.3), dict(window_half_frac=-1.0), dict(p2=1.5)]:
        with pytest.raises(T.TacticError) as ei:
            T.build_index(dev_bf16(K), dev_bf16(V), 16, 2, group_size=4, sampling=bad)
        assert ei.value.status == 1


# ----------------------------------------------------------------------------- boundary behaviour
def test_attention_only_before_any_selection_is_rejected(T):
    K, V, q = make_layer(1, 2, 4, 2048, seed=3)
    cents, asg, _ = oracle_layer_clustering(K, V, 32, 2, 3)
    index = T.import_index(dev_bf16(K), dev_bf16(V), cents, asg, group_size=4)
    out = torch.empty_like(dev_bf16(q))
    with pytest.raises(T.TacticError) as ei:
        T.decode_attention_only(dev_bf16(q), index, out)
    assert ei.value.status == 1
    T.decode(dev_bf16(q), index, 1.0)            # p = 1 runs no selection either
    with pytest.raises(T.TacticError):
        T.decode_attention_only(dev_bf16(q), index, out)
    ref = T.decode(dev_bf16(q), index, 0.9)
    T.decode_attention_only(dev_bf16(q), index, out)
    torch.cuda.synchronize()
    assert_same_decode(out, ref, "attention-only")


def test_selection_shared_memory_limit_is_reported_at_import(T):
    """G = 8 with C = 4096: the per-unit selection state exceeds one CTA's shared memory;
    the index is refused with UNSUPPORTED instead of failing every later decode."""
    n, C, G = 8192, 4096, 8
    rng = np.random.default_rng(0)
    K = (rng.standard_normal((1, 1, n, 128)) * 0.5).astype(np.float32)
    asg = (np.arange(n) % C).astype(np.int32)[None]
    cents = np.stack([K[0, 0][asg[0] == j].mean(0) for j in range(C)]).astype(np.float32)[None]
    with pytest.raises(T.TacticError) as ei:
        T.import_index(dev_bf16(K), dev_bf16(K), cents, asg, group_size=G)
    assert ei.value.status == 6
    T.import_index(dev_bf16(K), dev_bf16(K), cents, asg, group_size=4).close()   # G = 4 fits


def test_sharded_stages_with_tail_and_global_split(T):
    """Sequence-sharded stages (reading 23) with a recent-token tail appended to one shard
    and more units than CTAs / 2 (the attention kernel's global token split): the shard
    holding the tail attends it after its selected clusters, every unit is the LSE
    merge of the per-shard oracle parts."""
    B, H, G, S, n_shard, C, t = 10, 8, 4, 2, 1024, 16, 7
    units = B * H
    K, V, q = make_layer(B, H, G, S * n_shard, seed=61)
    rng = np.random.default_rng(61)
    from synth import bf16_round
    kt = bf16_round((rng.standard_normal((units, t, 128)) * 1.5).astype(np.float32))
    vt = bf16_round(rng.standard_normal((units, t, 128)).astype(np.float32))
    shard_idx, shard_o = [], []
    for s in range(S):
        sl = slice(s * n_shard, (s + 1) * n_shard)
        cents, asg, idxs = oracle_layer_clustering(K[:, :, sl], V[:, :, sl], C, 3, 61 + s)
        shard_idx.append(T.import_index(dev_bf16(K[:, :, sl]), dev_bf16(V[:, :, sl]), cents, asg, group_size=G))
        shard_o.append(idxs)
    T.append(shard_idx[1], dev_bf16(kt), dev_bf16(vt))        # the tail lives on shard 1
    qd = dev_bf16(q)
    p = 0.9
    lm = torch.stack([T.decode_stage1(qd, st).clone() for st in shard_idx])
    gmax = lm.max(dim=0).values
    mass = torch.stack([T.decode_stage1b(st, gmax).clone() for st in shard_idx]).sum(dim=0)
    parts = [T.decode_stage2(qd, st, p, gmax, mass) for st in shard_idx]
    o_parts = torch.stack([x[0].reshape(units * G, 128) for x in parts])
    l_parts = torch.stack([x[1].reshape(units * G) for x in parts])
    out = T.lse_merge(o_parts, l_parts).float().cpu().numpy().reshape(units, G, 128)
    for u in sorted({0, 1, units // 2, units - 1}):
        b, h = divmod(u, H)
        qo = q[b, h * G:(h + 1) * G]
        ro = O.decode_sharded(qo, [shard_o[s][u] for s in range(S)], p)
        op, lp = [], []
        for s in range(S):
            toks = O.cluster_tokens(shard_o[s][u], ro["unions"][s])
            Ks, Vs = shard_o[s][u].K, shard_o[s][u].V
            if s == 1:
                Ks, Vs = np.concatenate([Ks, kt[u]]), np.concatenate([Vs, vt[u]])
                toks = np.concatenate([toks, n_shard + np.arange(t)])
            o, l = O.sparse_attention(qo, Ks, Vs, toks)
            op.append(o)
            lp.append(l)
        ref, _ = O.lse_merge(np.array(op), np.array(lp))
        assert_output_close(out[u], ref, f"sharded + tail u={u}")
