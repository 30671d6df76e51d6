"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle on the same seeded
synthetic inputs.  Bars (BASELINE.json north_star): index sets bit-exact except within
1e-5 of the threshold; decode output max-abs <= 2e-2 and rel-L2 <= 5e-3; k-means
inertia within 1e-4 relative from an identical initialisation."""
import numpy as np
import pytest
import torch

from oracle import tactic_oracle as O
from synth import bf16_round, make_layer, make_unit, uniform_unit
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


def _layer(B, H, G, n, seed):
    K, V, q = make_layer(B, H, G, n, seed)
    return K, V, q


# ----------------------------------------------------------------------------- dense baseline
@pytest.mark.parametrize("B,H,G,n", [(1, 1, 4, 4096), (1, 2, 1, 1000), (2, 1, 8, 4133), (1, 3, 2, 777),
                                     (1, 1, 4, 64), (1, 1, 4, 1)])
def test_dense_decode_matches_full_attention(T, B, H, G, n):
    K, V, q = _layer(B, H, G, n, seed=n)
    Kd, Vd, qd = dev_bf16(K), dev_bf16(V), dev_bf16(q)
    lse = torch.empty((B, H * G), dtype=torch.float32, device="cuda")
    out = T.dense_decode(qd, Kd, Vd, lse=lse)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for b in range(B):
        for h in range(H):
            o, l = O.full_attention(q[b, h * G:(h + 1) * G], K[b, h], V[b, h])
            assert_output_close(got[b, h * G:(h + 1) * G], o, f"dense b{b} h{h}")
            np.testing.assert_allclose(lse[b, h * G:(h + 1) * G].cpu().numpy(), l, rtol=0, atol=2e-3)


@pytest.mark.parametrize("B,H,G,n,ctas", [(16, 8, 4, 333, 0),   # 128 units > CTAs/2: global split
                                          (2, 4, 4, 2000, 5),   # 8 units over 5 CTAs: several pieces per CTA
                                          (3, 2, 2, 517, 3)])
def test_dense_decode_global_split_epilogue(T, B, H, G, n, ctas):
    """Global token split: CTAs end several pieces, handed to the epilogue warp (combine,
    arrival, merge) while the consumers stream on; every unit against full attention."""
    K, V, q = _layer(B, H, G, n, seed=7 * n + B)
    lse = torch.empty((B, H * G), dtype=torch.float32, device="cuda")
    out = T.dense_decode(dev_bf16(q), dev_bf16(K), dev_bf16(V), lse=lse, num_ctas=ctas)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for b in range(B):
        for h in range(H):
            o, l = O.full_attention(q[b, h * G:(h + 1) * G], K[b, h], V[b, h])
            assert_output_close(got[b, h * G:(h + 1) * G], o, f"dense global b{b} h{h}")
            np.testing.assert_allclose(lse[b, h * G:(h + 1) * G].cpu().numpy(), l, rtol=0, atol=2e-3)


def test_dense_decode_strided_view(T):
    B, H, G, n = 1, 2, 4, 3000
    K, V, q = _layer(B, H, G, n, seed=5)
    big = torch.zeros((B, H, n + 100, 128), dtype=torch.bfloat16, device="cuda")
    big[:, :, :n] = dev_bf16(K)
    bigV = torch.zeros_like(big)
    bigV[:, :, :n] = dev_bf16(V)
    out = T.dense_decode(dev_bf16(q), big[:, :, :n], bigV[:, :, :n], num_ctas=37)
    got = out.float().cpu().numpy()
    for h in range(H):
        o, _ = O.full_attention(q[0, h * G:(h + 1) * G], K[0, h], V[0, h])
        assert_output_close(got[0, h * G:(h + 1) * G], o, "strided")


# ----------------------------------------------------------------------------- decode via imported clustering
def _import(T, K, V, cents, asg, G, **kw):
    return T.import_index(dev_bf16(K), dev_bf16(V), cents, asg, group_size=G, **kw)


def _check_unit_selection(res, u, G, heads_o, p, C):
    """order exact (ties by id), J within the threshold tolerance, union = union of the
    GPU prefixes of the oracle order."""
    for g in range(G):
        ho = heads_o[g]
        assert np.array_equal(res["order"][u, g], ho["order"]), f"order u{u} g{g}"
        Jg = int(res["J"][u, g])
        assert j_mismatch_allowed(ho, Jg, p), f"J u{u} g{g}: gpu {Jg} oracle {ho['J']}"
        fit = res["fit"][u, g]
        if not ho["fallback"]:
            assert fit[2] == pytest.approx(ho["m"], abs=2e-5)
            assert fit[4] == pytest.approx(ho["mu1"], rel=2e-5)
            assert fit[5] == pytest.approx(ho["mu2"], rel=2e-5)
            assert fit[0] == pytest.approx(ho["a"], rel=1e-4, abs=1e-6)
            assert fit[1] == pytest.approx(ho["b"], abs=1e-4 * max(abs(ho["mu1"]), 1e-12))
        assert fit[3] == pytest.approx(ho["W"], rel=1e-5)
    return True


@pytest.mark.parametrize("path", ["fused", "multi"])
@pytest.mark.parametrize("n,C,seed", [(4096, 64, 0), (4096, 64, 1), (32768, 256, 2), (5000, 77, 3)])
def test_import_decode_selection_and_output(T, n, C, seed, path):
    G = 4
    K, V, q = _layer(1, 2, G, n, seed)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 10, seed)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, T.OPT_CLUSTER_DECODE if path == "fused" else 0)
    assert (index.info()["select_cluster_size"] > 0) == (path == "fused")
    qd = dev_bf16(q)
    for p in [0.5, 0.8, 0.9, 0.95, 0.99]:
        res = T.decode_debug(qd, index, p)
        got = res["out"].float().cpu().numpy()
        for u in range(2):
            qo = q[0, u * G:(u + 1) * G]
            ro = O.decode_unit(qo, idxs[u], p)
            _check_unit_selection(res, u, G, ro["heads"], p, C)
            # union recomputed from the GPU's J on the oracle's order must equal the GPU union
            mask = np.zeros(C, dtype=bool)
            for g in range(G):
                pos = ro["heads"][g]["order"][:res["J"][u, g]]
                mask[pos[idxs[u].sizes[pos] > 0]] = True
            assert np.array_equal(mask, res["union_mask"][u]), f"union u{u} p{p}"
            # numerics against the oracle's attention over the GPU's union
            toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
            o, l = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
            assert_output_close(got[0, u * G:(u + 1) * G], o, f"out u{u} p{p}")
            np.testing.assert_allclose(res["lse"][0, u * G:(u + 1) * G].cpu().numpy(), l, atol=2e-3)


def test_import_decode_p1_equals_full_attention(T):
    G, n, C = 4, 4096, 64
    K, V, q = _layer(1, 2, G, n, 4)
    cents, asg, _ = oracle_layer_clustering(K, V, C, 10, 4)
    index = _import(T, K, V, cents, asg, G)
    out = T.decode(dev_bf16(q), index, 1.0).float().cpu().numpy()
    for u in range(2):
        o, _ = O.full_attention(q[0, u * G:(u + 1) * G], K[0, u], V[0, u])
        assert_output_close(out[0, u * G:(u + 1) * G], o, "p=1")


@pytest.mark.parametrize("path", ["fused", "multi"])
@pytest.mark.parametrize("G", [1, 2, 8])
def test_group_sizes(T, G, path):
    n, C = 4096, 64
    K, V, q = _layer(1, 1, G, n, 10 + G)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 10, G)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, T.OPT_CLUSTER_DECODE if path == "fused" else 0)
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    ro = O.decode_unit(q[0], idxs[0], 0.9)
    _check_unit_selection(res, 0, G, ro["heads"], 0.9, C)
    toks = O.cluster_tokens(idxs[0], np.nonzero(res["union_mask"][0])[0])
    o, _ = O.sparse_attention(q[0], idxs[0].K, idxs[0].V, toks)
    assert_output_close(res["out"].float().cpu().numpy()[0], o, f"G={G}")


@pytest.mark.parametrize("path", ["fused", "multi"])
def test_edge_cases_tiny_fallback_singletons_empty_clusters(T, path):
    opt = T.OPT_CLUSTER_DECODE if path == "fused" else 0
    G = 4
    # tiny n -> exact fallback (O6)
    u = make_unit(12, G, seed=1)
    K, V, q = u["K"][None, None], u["V"][None, None], u["q"][None]
    cents, asg, idxs = oracle_layer_clustering(K, V, 3, 10, 1)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, opt)
    for p in [0.5, 0.9]:
        res = T.decode_debug(dev_bf16(q), index, p)
        ro = O.decode_unit(q[0], idxs[0], p)
        assert ro["heads"][0]["fallback"]
        _check_unit_selection(res, 0, G, ro["heads"], p, 3)
    # C = n singleton clusters
    u = uniform_unit(256, G, seed=2)
    K, V, q = u["K"][None, None], u["V"][None, None], u["q"][None]
    idx = O.make_index(u["K"], u["V"], u["K"], np.arange(256))
    index = _import(T, K, V, u["K"][None], np.arange(256, dtype=np.int32)[None], G)
    T.set_options(index, opt)
    res = T.decode_debug(dev_bf16(q), index, 0.8)
    ro = O.decode_unit(q[0], idx, 0.8)
    _check_unit_selection(res, 0, G, ro["heads"], 0.8, 256)
    # empty clusters (ids 5, 17, 40 never assigned) and C = 1
    u = make_unit(3000, G, seed=3)
    K, V, q = u["K"][None, None], u["V"][None, None], u["q"][None]
    km = O.kmeans(u["K"], 48, 10, seed=3)
    asg = km["assign"].copy()
    remap = np.array([j for j in range(51) if j not in (5, 17, 40)])
    asg = remap[asg]
    cents = np.zeros((51, 128), dtype=np.float32)
    cents[remap] = km["centroids"].astype(np.float32)
    cents[[5, 17, 40]] = 1e3  # high criticality but empty: must never be selected
    idx = O.make_index(u["K"], u["V"], cents, asg)
    index = _import(T, K, V, cents[None], asg.astype(np.int32)[None], G)
    T.set_options(index, opt)
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    ro = O.decode_unit(q[0], idx, 0.9)
    _check_unit_selection(res, 0, G, ro["heads"], 0.9, 51)
    assert not res["union_mask"][0][[5, 17, 40]].any()
    index1 = _import(T, K, V, u["K"][:1][None], np.zeros((1, 3000), dtype=np.int32), G)
    T.set_options(index1, opt)
    out1 = T.decode(dev_bf16(q), index1, 0.5).float().cpu().numpy()
    o, _ = O.full_attention(q[0], u["K"], u["V"])
    assert_output_close(out1[0], o, "C=1")


def test_invalid_arguments(T):
    K, V, q = _layer(1, 1, 4, 512, 0)
    index = T.build_index(dev_bf16(K), dev_bf16(V), 8, 2, group_size=4)
    for bad in [0.0, -0.1, 1.5, float("nan")]:
        with pytest.raises(T.TacticError) as ei:
            T.decode(dev_bf16(q), index, bad)
        assert ei.value.status == 1
    with pytest.raises(T.TacticError):
        T.build_index(dev_bf16(K), dev_bf16(V), 513, 2)
    with pytest.raises(T.TacticError):
        T.build_index(dev_bf16(K), dev_bf16(V), 8, 0)
    Kn = K.copy()
    Kn[0, 0, 7, 3] = np.nan
    with pytest.raises(T.TacticError) as ei:
        T.build_index(dev_bf16(Kn), dev_bf16(V), 8, 2, flags=T.FLAG_VALIDATE)
    assert ei.value.status == 5


# ----------------------------------------------------------------------------- k-means build
@pytest.mark.parametrize("n,C,seed", [(4096, 64, 0), (32768, 256, 1), (10000, 100, 2)])
def test_gpu_kmeans_inertia_parity(T, n, C, seed):
    K, V, q = _layer(1, 2, 4, n, seed)
    units = 2
    init = np.stack([O.init_indices(n, C, seed, u) for u in range(units)]).astype(np.int32)
    index = T.build_index(dev_bf16(K), dev_bf16(V), C, 10, group_size=4, init=init)
    ex = index.export()
    for u in range(units):
        km = O.kmeans(K[0, u], C, 10, init=init[u])
        assert ex["inertia"][u] == pytest.approx(km["inertia"], rel=1e-4), f"unit {u}"
        assert 1 <= ex["iters_run"][u] <= 10
        # structural: centroids are float32 means of the exported assignment
        a = ex["assign"][u]
        for j in np.unique(a)[:20]:
            np.testing.assert_allclose(ex["centroids"][u, j], K[0, u][a == j].astype(np.float64).mean(0),
                                       rtol=1e-6, atol=1e-6)


def test_gpu_kmeans_sampler_matches_oracle_sampler(T):
    # same SplitMix64/Fisher-Yates init on both sides -> same trajectory (1 iteration)
    n, C = 4096, 64
    K, V, q = _layer(1, 1, 4, n, 7)
    index = T.build_index(dev_bf16(K), dev_bf16(V), C, 1, group_size=4, seed=11)
    ex = index.export()
    km = O.kmeans(K[0, 0], C, 1, seed=11, unit=0)
    assert ex["inertia"][0] == pytest.approx(km["inertia"], rel=1e-5)
    assert np.mean(ex["assign"][0] == km["assign"]) > 0.999


def test_tcgen05_assignment_matches_simt_kernel(T):
    n, C = 8192, 256
    K, V, q = _layer(1, 1, 4, n, 8)
    init = O.init_indices(n, C, 8, 0)[None].astype(np.int32)
    a_tc = T.build_index(dev_bf16(K), dev_bf16(V), C, 1, init=init).export()["assign"]
    a_si = T.build_index(dev_bf16(K), dev_bf16(V), C, 1, init=init, flags=T.FLAG_KMEANS_SIMT).export()["assign"]
    assert np.mean(a_tc == a_si) > 0.999
    a_o = O.kmeans(K[0, 0], C, 1, init=init[0])["assign"]
    assert np.mean(a_tc[0] == a_o) > 0.999


def test_build_then_decode_p1_full_attention(T):
    G, n, C = 4, 8192, 64
    K, V, q = _layer(2, 2, G, n, 9)
    index = T.build_index(dev_bf16(K), dev_bf16(V), C, 10, group_size=G, seed=3)
    out = T.decode(dev_bf16(q), index, 1.0).float().cpu().numpy()
    out9 = T.decode(dev_bf16(q), index, 0.9).float().cpu().numpy()
    for b in range(2):
        for h in range(2):
            sl = slice(h * G, (h + 1) * G)
            o, _ = O.full_attention(q[b, sl], K[b, h], V[b, h])
            assert_output_close(out[b, sl], o, "build p=1")
            assert np.all(np.isfinite(out9[b, sl]))


# ----------------------------------------------------------------------------- misc paths
def test_lse_merge_kernel(T):
    rng = np.random.default_rng(0)
    S, R = 5, 37
    o = rng.standard_normal((S, R, 128)).astype(np.float32)
    l = (rng.standard_normal((S, R)) * 3).astype(np.float32)
    l[2, 4] = -np.inf
    out = T.lse_merge(torch.from_numpy(o).cuda(), torch.from_numpy(l).cuda()).float().cpu().numpy()
    ref, _ = O.lse_merge(o, l)
    assert_output_close(out, ref, "lse_merge")


def test_decode_host_and_graph_capture(T):
    G, n, C = 4, 4096, 64
    K, V, q = _layer(1, 2, G, n, 12)
    cents, asg, _ = oracle_layer_clustering(K, V, C, 5, 12)
    index = _import(T, K, V, cents, asg, G)
    qd = dev_bf16(q)
    ref = T.decode(qd, index, 0.9)
    torch.cuda.synchronize()
    host = T.decode_host(qd.cpu(), index, 0.9)          # pageable: copies in and out
    assert_same_decode(host, ref, "host-buffer decode")
    q_pin = qd.cpu().pin_memory()                          # pinned + mapped: zero-copy path
    o_pin = torch.empty_like(q_pin).pin_memory()
    for _ in range(3):                                     # capture, then graph replays
        o_pin.zero_()
        T.decode_host(q_pin, index, 0.9, o_pin)
        assert_same_decode(o_pin, ref, "zero-copy host decode")
    q_pin.copy_((qd * 0.5).cpu())                          # new contents, same buffers
    T.decode_host(q_pin, index, 0.9, o_pin)
    assert_same_decode(o_pin, T.decode(qd * 0.5, index, 0.9), "zero-copy host decode, new q")
    T.set_options(index, T.OPT_DETERMINISTIC)  # the partial merge: bit-identical entry points
    ref = T.decode(qd, index, 0.9)
    torch.cuda.synchronize()
    host = T.decode_host(qd.cpu(), index, 0.9)
    assert torch.equal(host, ref.cpu())
    T.decode_host(q_pin.copy_(qd.cpu()), index, 0.9, o_pin)
    assert torch.equal(o_pin, ref.cpu())
    out = torch.empty_like(qd)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        T.decode(qd, index, 0.9, out=out)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        T.decode(qd, index, 0.9, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_sharded_stages_match_sharded_oracle(T):
    G, S, n_shard, C = 4, 4, 4096, 64
    u = make_unit(S * n_shard, G, seed=21)
    q = u["q"]
    shards_o, st = [], []
    for s in range(S):
        sl = slice(s * n_shard, (s + 1) * n_shard)
        Ks, Vs = u["K"][sl], u["V"][sl]
        idx, km = O.build_index(Ks, Vs, C, 10, seed=21, unit=s)
        shards_o.append(idx)
        st.append(_import(T, Ks[None, None], Vs[None, None], km["centroids"].astype(np.float32)[None],
                          km["assign"].astype(np.int32)[None], G))
    qd = dev_bf16(q[None])
    for p in [0.5, 0.9, 1.0]:
        ro = O.decode_sharded(q, shards_o, p)
        lm = torch.stack([T.decode_stage1(qd, st[s]).clone() for s in range(S)])
        gmax = lm.max(dim=0).values
        mass = torch.stack([T.decode_stage1b(st[s], gmax).clone() for s in range(S)]).sum(dim=0)
        parts = [T.decode_stage2(qd, st[s], p, gmax, mass) for s in range(S)]
        o_parts = torch.stack([x[0].reshape(G, 128) for x in parts])
        l_parts = torch.stack([x[1].reshape(G) for x in parts])
        out = T.lse_merge(o_parts, l_parts).float().cpu().numpy()
        for g in range(G):
            assert float(gmax[0, g, 0]) == pytest.approx(ro["m_glob"][g], abs=2e-5)
            assert float(gmax[0, g, 1]) == pytest.approx(ro["theta_max"][g], rel=1e-12)
            np.testing.assert_allclose(mass[0, g].cpu().numpy(), ro["mass_total"][g], rtol=1e-4, atol=1e-12)
        assert_output_close(out, ro["o"], f"sharded p={p}")


# ----------------------------------------------------------------------------- full size (C2 launch config)
@pytest.mark.slow
def test_c2_full_size_sampled_parity(T):
    """C2 shape (Llama-3-8B layer, 128K, 8 units) in the bench's launch configuration.
    The oracle clustering (3 Lloyd iterations to bound CPU time) is imported; every unit's
    selection and output is checked against the oracle."""
    G, n, C = 4, 131072, 1024
    K, V, q = _layer(1, 8, G, n, 0)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 0)
    index = _import(T, K, V, cents, asg, G)
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    got = res["out"].float().cpu().numpy()
    for u in range(8):
        qo = q[0, u * G:(u + 1) * G]
        ro = O.decode_unit(qo, idxs[u], 0.9)
        _check_unit_selection(res, u, G, ro["heads"], 0.9, C)
        toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
        o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
        assert_output_close(got[0, u * G:(u + 1) * G], o, f"C2 unit {u}")
    # p = 1 through the same index equals full attention (sampled units)
    out1 = T.decode(dev_bf16(q), index, 1.0).float().cpu().numpy()
    for u in (0, 5):
        o, _ = O.full_attention(q[0, u * G:(u + 1) * G], K[0, u], V[0, u])
        assert_output_close(out1[0, u * G:(u + 1) * G], o, f"C2 p=1 unit {u}")


# ----------------------------------------------------------------------------- attention work-split modes
@pytest.mark.parametrize("B,H,n,C", [(12, 8, 2048, 32),    # 96 units > CTAs/2: global token split,
                                     (64, 8, 1024, 16),    # C3-like unit count (512 units)
                                     (7, 10, 2048, 32),    # 70 units <= CTAs/2: unit-aligned split with
                                     (9, 8, 4096, 64)])    # 1-3 CTAs per unit (designated merger alone)
def test_global_split_many_units(T, B, H, n, C):
    """More units than half the CTAs (BASELINE configs[2] shape class: batch x KV heads):
    the fit kernel's last unit writes the token prefix over units and the attention
    kernel cuts one global token list (a CTA may hold pieces of two units).  Just below
    that (70 / 72 units) the unit-aligned split gives units 1-3 CTAs, so the designated
    merger of the reference-shift merge often has no other piece to wait for."""
    G = 4
    K, V, q = _layer(B, H, G, n, 500 + B)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, B)
    index = _import(T, K, V, cents, asg, G)
    units = B * H
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    got = res["out"].float().cpu().numpy()
    for u in sorted({0, 1, units // 3, units // 2, units - 2, units - 1}):
        b, h = divmod(u, H)
        qo = q[b, h * G:(h + 1) * G]
        ro = O.decode_unit(qo, idxs[u], 0.9)
        _check_unit_selection(res, u, G, ro["heads"], 0.9, C)
        toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
        o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
        assert_output_close(got[b, h * G:(h + 1) * G], o, f"units={units} u={u}")


def test_unit_split_per_unit_list_fallback(T):
    """Unit-aligned split whose units' work lists do not all fit the attention kernel's
    shared-memory list area (8 units x C = 2048): the CTA stages its own unit's list."""
    G, n, C = 4, 16384, 2048
    K, V, q = _layer(1, 8, G, n, 901)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 2, 901)
    index = _import(T, K, V, cents, asg, G)
    for p in (0.9, 1.0):
        res = T.decode_debug(dev_bf16(q), index, p)
        got = res["out"].float().cpu().numpy()
        for u in (0, 3, 7):
            qo = q[0, u * G:(u + 1) * G]
            if p < 1.0:
                ro = O.decode_unit(qo, idxs[u], p)
                _check_unit_selection(res, u, G, ro["heads"], p, C)
                toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
                o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
            else:
                o, _ = O.full_attention(qo, K[0, u], V[0, u])
            assert_output_close(got[0, u * G:(u + 1) * G], o, f"C={C} p={p} u={u}")


# ----------------------------------------------------------------------------- NEXT 1: multi-step generation
def _tail_tokens(units, t, seed):
    rng = np.random.default_rng(seed)
    kt = bf16_round((rng.standard_normal((units, t, 128)) * 1.5).astype(np.float32))
    vt = bf16_round(rng.standard_normal((units, t, 128)).astype(np.float32))
    return kt, vt


@pytest.mark.parametrize("path", ["multi", "fused"])
@pytest.mark.parametrize("B,H,n,C", [(1, 2, 4096, 64),     # unit-aligned split
                                     (12, 8, 2048, 32)])   # global token split (96 units)
def test_tail_append_decode_parity(T, B, H, n, C, path):
    """Appended tokens (two appends) are attended in full after the selected clusters;
    the selection itself is unchanged (it ranks the clustered tokens only)."""
    G = 4
    K, V, q = _layer(B, H, G, n, 700 + B)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, B)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, T.OPT_CLUSTER_DECODE if path == "fused" else 0)
    units = B * H
    kt1, vt1 = _tail_tokens(units, 21, 1)
    kt2, vt2 = _tail_tokens(units, 44, 2)
    T.append(index, dev_bf16(kt1), dev_bf16(vt1))
    T.append(index, dev_bf16(kt2), dev_bf16(vt2))
    assert T.tail_info(index)[0] == 65
    kt, vt = np.concatenate([kt1, kt2], axis=1), np.concatenate([vt1, vt2], axis=1)
    qd = dev_bf16(q)
    for p in (0.9, 1.0):
        res = T.decode_debug(qd, index, p)
        got = res["out"].float().cpu().numpy()
        for u in sorted({0, 1, units // 2, units - 1}):
            b, h = divmod(u, H)
            qo = q[b, h * G:(h + 1) * G]
            if p < 1.0:
                ro = O.decode_unit(qo, idxs[u], p)
                _check_unit_selection(res, u, G, ro["heads"], p, C)
                toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
                K_all = np.concatenate([K[b, h], kt[u]])
                V_all = np.concatenate([V[b, h], vt[u]])
                o, _ = O.sparse_attention(qo, K_all, V_all, np.concatenate([toks, n + np.arange(65)]))
            else:
                o, _ = O.full_attention(qo, np.concatenate([K[b, h], kt[u]]), np.concatenate([V[b, h], vt[u]]))
            assert_output_close(got[b, h * G:(h + 1) * G], o, f"tail p={p} u={u}")


def test_tail_capacity_and_errors(T):
    G, n, C = 4, 1024, 16
    K, V, q = _layer(1, 1, G, n, 3)
    cents, asg, _ = oracle_layer_clustering(K, V, C, 2, 3)
    index = _import(T, K, V, cents, asg, G)
    T.set_tail_capacity(index, 8)
    assert T.tail_info(index) == (0, 8)
    kt, vt = _tail_tokens(1, 5, 4)
    T.append(index, dev_bf16(kt), dev_bf16(vt))
    with pytest.raises(T.TacticError):        # 5 + 5 > 8: the caller must re-cluster
        T.append(index, dev_bf16(kt), dev_bf16(vt))
    with pytest.raises(T.TacticError):        # capacity changes need an empty tail
        T.set_tail_capacity(index, 16)
    assert T.tail_info(index) == (5, 8)


def test_assign_tokens_matches_oracle(T):
    """SPEC assign_token: nearest float32 centroid of new keys, float64."""
    G, n, C = 4, 8192, 128
    K, V, q = _layer(1, 4, G, n, 12)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 12)
    index = _import(T, K, V, cents, asg, G)
    kt, _ = _tail_tokens(4, 300, 12)
    kt[:, :50] = K[0, :, 1000:1050]            # keys resembling the cache
    got = T.assign_tokens(index, dev_bf16(kt)).cpu().numpy()
    for u in range(4):
        ref = O.assign_tokens(kt[u], cents[u].astype(np.float64))
        d = ((kt[u][:, None, :].astype(np.float64) - cents[u][None].astype(np.float64)) ** 2).sum(-1)
        for i in np.nonzero(got[u] != ref)[0]:   # only exact-arithmetic near-ties may differ
            assert abs(d[i, got[u][i]] - d[i, ref[i]]) <= 1e-9 * d[i, ref[i]], (u, i)


def test_decode_session_reclusters_and_matches_full_attention(T):
    """DecodeSession: append -> decode each step; a full tail triggers re-clustering of
    the whole cache.  At p = 1 every step equals full attention over all tokens so far."""
    G, n, C, H = 4, 2048, 32, 2
    K, V, q = _layer(1, H, G, n, 21)
    Kd, Vd = dev_bf16(K), dev_bf16(V)
    s = T.DecodeSession(Kd, Vd, C, 3, group_size=G, tail_capacity=6)
    K_all, V_all = K.copy(), V.copy()
    for step in range(15):
        kt, vt = _tail_tokens(H, 1, 100 + step)
        qs = bf16_round(np.random.default_rng(step).standard_normal((1, H * G, 128)).astype(np.float32))
        out = s.step(dev_bf16(qs), dev_bf16(kt), dev_bf16(vt), 1.0).float().cpu().numpy()
        K_all = np.concatenate([K_all, kt[None]], axis=2)
        V_all = np.concatenate([V_all, vt[None]], axis=2)
        for h in range(H):
            o, _ = O.full_attention(qs[0, h * G:(h + 1) * G], K_all[0, h], V_all[0, h])
            assert_output_close(out[0, h * G:(h + 1) * G], o, f"step {step} h {h}")
    assert s.rebuilds == 2 and s.seq_len == n + 15


# ----------------------------------------------------------------------------- NEXT 3: Table-1 diagnostics
def test_exact_logits_and_table1_match_oracle(T):
    """tactic_exact_logits (layout order) and tools/table1.py against the oracle's
    optimal_budget / cluster_optimal_budget / cumulative_score per head."""
    import sys
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    from tools.table1 import table1_stats
    G, n, C = 4, 4096, 64
    K, V, q = _layer(1, 2, G, n, 31)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 31)
    index = _import(T, K, V, cents, asg, G)
    qd = dev_bf16(q)
    lg = T.exact_logits(qd, index).cpu().numpy()
    for u in range(2):
        ref = (idxs[u].K[idxs[u].perm] @ q[0, u * G:(u + 1) * G].T.astype(np.float64)) / np.sqrt(128)
        np.testing.assert_allclose(lg[u].T, ref, atol=2e-4, rtol=1e-5)
    sizes = np.stack([idxs[u].sizes for u in range(2)])
    st = table1_stats(T, qd, index, sizes, [0.5, 0.9])
    for p in (0.5, 0.9):
        ph = st[str(p)]["_per_head"]
        res = T.decode_debug(qd, index, p)
        for u in range(2):
            for g in range(G):
                qg = q[0, u * G + g]
                assert abs(ph["optimal"][u, g] - O.optimal_budget(qg, idxs[u].K, p)) <= 1
                assert abs(ph["cluster_optimal"][u, g] - O.cluster_optimal_budget(qg, idxs[u], p)) <= \
                    idxs[u].sizes.max()
                own = res["order"][u, g][:res["J"][u, g]]
                toks = O.cluster_tokens(idxs[u], own)
                assert ph["tactic_own"][u, g] == len(toks)
                assert ph["achieved_own"][u, g] == pytest.approx(O.cumulative_score(qg, idxs[u].K, toks), abs=1e-5)


# ----------------------------------------------------------------------------- NEXT 2: per-head loading ablation
def test_per_head_loading_matches_oracle_own_set_attention(T):
    """tactic_decode_per_head: every head attends only its own S_g (P:695 ablation; SPEC
    own-set normalisation S:421), against the oracle's decode_unit_per_head."""
    G, n, C = 4, 8192, 128
    K, V, q = _layer(1, 3, G, n, 41)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 41)
    index = _import(T, K, V, cents, asg, G)
    qd = dev_bf16(q)
    for p in (0.5, 0.9):
        got = T.decode_per_head(qd, index, p).float().cpu().numpy()
        res = T.decode_debug(qd, index, p)
        for u in range(3):
            qo = q[0, u * G:(u + 1) * G]
            ro = O.decode_unit_per_head(qo, idxs[u], p)
            for g in range(G):   # compare only heads whose selection matches exactly
                if int(res["J"][u, g]) == ro["heads"][g]["J"]:
                    assert_output_close(got[0, u * G + g:u * G + g + 1], ro["o"][g:g + 1], f"p={p} u={u} g={g}")


# ----------------------------------------------------------------------------- NEXT 4: fixed-budget baseline
@pytest.mark.parametrize("path", ["multi", "fused"])
def test_fixed_budget_selection_and_output(T, path):
    G, n, C = 4, 8192, 128
    K, V, q = _layer(1, 2, G, n, 51)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 51)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, T.OPT_CLUSTER_DECODE if path == "fused" else 0)
    qd = dev_bf16(q)
    for budget in (100, 700):
        out, J = T.decode_fixed_budget(qd, index, budget)
        ph, J2 = T.decode_fixed_budget(qd, index, budget, per_head=True)
        assert np.array_equal(J, J2)
        got, gph = out.float().cpu().numpy(), ph.float().cpu().numpy()
        for u in range(2):
            qo = q[0, u * G:(u + 1) * G]
            mask = np.zeros(C, dtype=bool)
            for g in range(G):
                r = O.fixed_budget_select(qo[g], idxs[u], budget)
                assert J[u, g] == r["J"], (budget, u, g)
                mask[r["S"]] = True
                o_own, _ = O.sparse_attention(qo[g], idxs[u].K, idxs[u].V, O.cluster_tokens(idxs[u], r["S"]))
                assert_output_close(gph[0, u * G + g:u * G + g + 1], o_own, f"own b={budget} u={u} g={g}")
            o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, O.cluster_tokens(idxs[u], np.nonzero(mask)[0]))
            assert_output_close(got[0, u * G:(u + 1) * G], o, f"union b={budget} u={u}")


def test_fig5_variance_tool_runs_and_is_consistent(T):
    """tools/table1.fig5_variance: the fixed budget matches Tactic's mean token count;
    eps of every head obeys the Appendix-A bound eps <= 2 (1 - p(I)) max |v|."""
    import sys
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    from tools.table1 import fig5_variance
    G, n, C = 4, 8192, 128
    K, V, q = _layer(1, 4, G, n, 61)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 61)
    index = _import(T, K, V, cents, asg, G)
    r = fig5_variance(T, dev_bf16(q), index, np.stack([i.sizes for i in idxs]), dev_bf16(K), dev_bf16(V), 0.9)
    vmax = float(np.max(np.linalg.norm(V.reshape(-1, 128), axis=1)))
    for k in ("tactic", "fixed_budget"):
        assert r[k]["eps"]["max"] <= 2 * (1 - r[k]["achieved_p"]["min"]) * vmax + 2e-2
    assert abs(r["fixed_budget"]["tokens"]["mean"] - r["tactic"]["tokens"]["mean"]) <= 0.5 * r["tactic"]["tokens"]["mean"] + 200


def test_windows_exact_variant_matches_oracle(T):
    G, n, C = 4, 32768, 256
    K, V, q = _layer(1, 2, G, n, 71)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 71)
    index = _import(T, K, V, cents, asg, G)
    T.set_options(index, T.OPT_WINDOWS_EXACT)
    qd = dev_bf16(q)
    for p in (0.5, 0.9, 0.99):
        res = T.decode_debug(qd, index, p)
        for u in range(2):
            ro = O.decode_unit(q[0, u * G:(u + 1) * G], idxs[u], p, windows_exact=True)
            _check_unit_selection(res, u, G, ro["heads"], p, C)
    T.set_options(index, 0)
    res = T.decode_debug(qd, index, 0.9)
    ro = O.decode_unit(q[0, 0:G], idxs[0], 0.9)
    _check_unit_selection(res, 0, G, ro["heads"], 0.9, C)


def test_per_head_loading_with_tail(T):
    """Per-head loading (G = 1 work units reading unit u / G) attends its own clusters plus
    the whole recent-token tail of its KV unit."""
    G, n, C = 4, 4096, 64
    K, V, q = _layer(1, 2, G, n, 81)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 81)
    index = _import(T, K, V, cents, asg, G)
    kt, vt = _tail_tokens(2, 29, 81)
    T.append(index, dev_bf16(kt), dev_bf16(vt))
    got = T.decode_per_head(dev_bf16(q), index, 0.9).float().cpu().numpy()
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    for u in range(2):
        qo = q[0, u * G:(u + 1) * G]
        ro = O.decode_unit_per_head(qo, idxs[u], 0.9)
        for g in range(G):
            if int(res["J"][u, g]) != ro["heads"][g]["J"]:
                continue
            toks = np.concatenate([O.cluster_tokens(idxs[u], ro["heads"][g]["S"]), n + np.arange(29)])
            o, _ = O.sparse_attention(qo[g], np.concatenate([K[0, u], kt[u]]), np.concatenate([V[0, u], vt[u]]), toks)
            assert_output_close(got[0, u * G + g:u * G + g + 1], o, f"u={u} g={g}")


def test_attention_only_reproduces_decode(T):
    """tactic_decode_attention_only reruns S8 + S9 (the multi-kernel attention kernel) over
    the work lists of the last selection: bit-identical to the multi-kernel decode, also
    when called repeatedly; the one-launch decode writes the same lists (its own token
    split, so equal within rounding)."""
    B, H, G, n, C = 1, 2, 4, 8192, 64
    K, V, q = _layer(B, H, G, n, 321)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, B)
    index = _import(T, K, V, cents, asg, G)
    qd = dev_bf16(q)
    for opt in (T.OPT_DETERMINISTIC, 0, T.OPT_CLUSTER_DECODE):
        T.set_options(index, opt)
        ref = T.decode(qd, index, 0.9)
        out = torch.empty_like(ref)
        for _ in range(3):
            out.zero_()
            T.decode_attention_only(qd, index, out)
            torch.cuda.synchronize()
            if opt == T.OPT_DETERMINISTIC:
                assert torch.equal(out, ref)
            elif opt == 0:
                assert_same_decode(out, ref, "attention-only")
            else:
                assert_output_close(out.float().cpu().numpy(), ref.float().cpu().numpy(), "attention-only")


@pytest.mark.parametrize("sel_scale,att_scale", [(1.0, 30.0), (30.0, 1.0), (1.0, 1.0)])
def test_reference_shift_merge_window_and_fallback(T, sel_scale, att_scale):
    """S9 by the reference shift (attention.cu): every piece adds 2^(m_c - m_ref) (o_c, l_c)
    with m_ref = the fit's sampled max logit.  Attention-only over the last selection's
    lists with a query whose logits sit far above (x30) or below (selection at x30) that
    shift leaves the fp32 window, so the merging CTA must fall back to the partial merge;
    in every case the output equals the oracle's attention over the same union, and the
    deterministic option gives the same result within rounding."""
    B, H, G, n, C = 1, 8, 4, 16384, 128
    K, V, q = _layer(B, H, G, n, 4242)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 4242)
    index = _import(T, K, V, cents, asg, G)
    q_sel = bf16_round(q * sel_scale)
    q_att = bf16_round(q * att_scale)
    res = T.decode_debug(dev_bf16(q_sel), index, 0.9)   # selection -> union lists + m_ref
    out = torch.empty_like(dev_bf16(q_att))
    T.decode_attention_only(dev_bf16(q_att), index, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for u in range(B * H):
        toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
        o_ref, _ = O.sparse_attention(q_att.reshape(B * H, G, 128)[u], idxs[u].K, idxs[u].V, toks)
        assert_output_close(got.reshape(B * H, G, 128)[u], o_ref, f"unit {u} scales {sel_scale}/{att_scale}")
    T.set_options(index, T.OPT_DETERMINISTIC)
    T.decode_debug(dev_bf16(q_sel), index, 0.9)
    out2 = torch.empty_like(out)
    T.decode_attention_only(dev_bf16(q_att), index, out2)
    torch.cuda.synchronize()
    assert_output_close(out2.float().cpu().numpy(), got, "deterministic vs reference-shift merge")


@pytest.mark.parametrize("num_ctas", [64, 300])
def test_reference_shift_merge_protocols(T, num_ctas):
    """The reference-shift merge with the designated merger (grid fits the device: 64 CTAs)
    and with the last-arriver atomic (300 CTAs > SMs: a polling CTA could hold an SM that a
    CTA it waits for needs, so the library falls back): both match the oracle and each
    other."""
    B, H, G, n, C = 1, 8, 4, 16384, 128
    K, V, q = _layer(B, H, G, n, 77)
    cents, asg, idxs = oracle_layer_clustering(K, V, C, 3, 77)
    index = _import(T, K, V, cents, asg, G, num_ctas=num_ctas)
    res = T.decode_debug(dev_bf16(q), index, 0.9)
    got = res["out"].float().cpu().numpy()
    for u in (0, 3, 7):
        qo = q[0, u * G:(u + 1) * G]
        toks = O.cluster_tokens(idxs[u], np.nonzero(res["union_mask"][u])[0])
        o, _ = O.sparse_attention(qo, idxs[u].K, idxs[u].V, toks)
        assert_output_close(got[0, u * G:(u + 1) * G], o, f"num_ctas={num_ctas} u={u}")
