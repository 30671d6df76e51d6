#!/usr/bin/env python
"""bench.py -- Tactic decode-attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--p 0.9]

A *step* is one decode layer-step of the whole hot path (S1-S9: centroid scoring, cluster
sort, sampled exact scoring, a/x+b fit, estimated-mass selection, GQA union + work list,
split-KV flash-decode, LSE merge) over one C2 layer: Llama-3-8B shape (32 Q / 8 KV
heads, d=128), 128K context, batch 1, 1024 clusters per KV head, p=0.9, bf16 KV.
The index (tcgen05 k-means + cluster-contiguous relayout) is built once per layer and
timed separately ("build").  N>1 (torchrun): each rank runs its own batch-1 C2 layer
(batch x KV-head sharding, no collective on the data path), scaling "weak"; the
reported time is the max over ranks divided by N (job-level us per layer-step).

Layers: the timed steps cycle over LAYERS = 8 distinct synthetic layers (seeds 8 rank + l),
one index each, as a model's decode does (>= 8 distinct layer caches); the
selected fraction varies from layer to layer, so the mean is over layers.
L2: a 256 MiB buffer is written before every timed step as well (the sparse working set
would otherwise partly stay in the 126 MB L2); each step is bracketed by CUDA events on
the launching stream.  --impl reference times the float64 CPU oracle (the reference arm of
this tier) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attn µs/layer-step & HBM GB/s vs own dense decode @128K, p=0.9, 1/2/4/8 GPU"
UNIT = "µs/layer-step"
WORKLOAD = "C2"
CFG = dict(B=1, Hkv=8, G=4, n=131072, C=1024, iters=10)
LAYERS = 8
PAPER_CONTEXT = ("paper (context, not target): up to 7.29x decode-attention and 1.58x end-to-end speedup vs "
                 "FlashInfer full attention on Nvidia Ada 6000, CUDA 12.4 (P:47, P:404, P:691, P:701)")


def _config(args, n_gpus):
    return {"workload": f"{WORKLOAD}: Llama-3-8B layer (32 Q / 8 KV heads, d=128), 128K context, batch 1 per GPU, "
                        f"1024 clusters/KV head, p={args.p}",
            "global_batch": n_gpus, "seq_len": CFG["n"], "n_clusters": CFG["C"], "p": args.p,
            "parallelism": f"batch x KV-head sharded over {n_gpus} GPU(s), no data-path collective",
            "l2": "cold L2 before every timed step: 256 MiB buffer written, then a 256 MiB buffer read (write-back drained); "
                  "within a step each layer reads its own K/V (512 MB per layer > L2)",
            "step": f"one decode step through all {LAYERS} synthetic layers, one CUDA graph, layers serialised "
                    f"(no cross-layer overlap); value = step time / {LAYERS}",
            "inputs": f"tactic-synth-v1 (synth/), {LAYERS} layers per GPU (seeds {LAYERS} rank + l)"}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks (NVML sampling thread)
class ClockSampler:
    def __init__(self, dev_index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.period = period_s

    def _run(self):
        nv = self.nv
        names = {}
        for attr in ("nvmlClocksEventReasonHwSlowdown", "nvmlClocksEventReasonHwThermalSlowdown",
                     "nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksEventReasonSwPowerCap",
                     "nvmlClocksEventReasonHwPowerBrakeSlowdown"):
            if hasattr(nv, attr):
                names[getattr(nv, attr)] = attr.replace("nvmlClocksEventReason", "")
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ byte model
def step_bytes(dbg, sizes, G, n, C):
    """Algorithmic bytes of one layer-step: fp32 centroids, sampled K rows not re-read by the
    attention, selected (union) K+V rows, q/out, from the selection the GPU actually made."""
    from paper_2502_12216_b200.tactic import sample_constants
    sc = sample_constants(n)
    units = sizes.shape[0]
    tot_union, tot_sampled_extra = 0, 0
    for u in range(units):
        off = np.concatenate([[0], np.cumsum(sizes[u])])
        um = dbg["union_mask"][u]
        tot_union += int(sizes[u][um].sum())
        rows = set()
        if sc["fallback"]:
            continue
        ranks = np.concatenate([np.arange(1, sc["N"] + 1), np.arange(sc["x1"] - sc["w"], sc["x1"] + sc["w"] + 1),
                                np.arange(sc["x2"] - sc["w"], sc["x2"] + sc["w"] + 1)])
        for g in range(G):
            order = dbg["order"][u, g]
            ends = np.cumsum(sizes[u][order])
            r = np.searchsorted(ends, ranks, side="left")
            cid = order[r]
            start = ends[r] - sizes[u][cid]
            row = off[cid] + (ranks - 1 - start)
            sel = ~um[cid]
            rows.update(row[sel].tolist())
        tot_sampled_extra += len(rows)
    cent = units * C * 128 * 4
    qo = 2 * units * G * 128 * 2
    attn = tot_union * 128 * 2 * 2
    return {"centroids": cent, "sampled_k_extra": tot_sampled_extra * 256, "union_kv": attn, "q_out": qo,
            "total": cent + tot_sampled_extra * 256 + attn + qo, "union_tokens": tot_union,
            "union_frac": tot_union / (units * n)}


# ------------------------------------------------------------------ reference arm (oracle on CPU)
def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import tactic_oracle as O
    from synth import make_unit
    threads = _cpu_threads()
    u = make_unit(CFG["n"], CFG["G"], seed=0, b=0, h=0)
    idx, _ = O.build_index(u["K"], u["V"], CFG["C"], 1, seed=0, unit=0)   # setup, untimed
    for _ in range(args.warmup):
        O.decode_unit(u["q"], idx, args.p)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.decode_unit(u["q"], idx, args.p)
        ts.append(time.perf_counter() - t0)
    per_unit = float(np.mean(ts))
    val = per_unit * CFG["B"] * CFG["Hkv"] * 1e6          # one layer-step = 8 units
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": val / 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": _config(args, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"1 of 8 units per step (KV head 0, n=131072, C=1024; index from 1 oracle "
                                       f"Lloyd iteration, untimed), scaled x8 to a layer-step"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            return int(max(i.get("num_threads", 1) for i in info))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


def cpu_baseline(args, budget_s=12.0):
    """Time the oracle decode (as it stands) on a bounded sample of the C2 workload."""
    from oracle import tactic_oracle as O
    from synth import make_unit
    u = make_unit(CFG["n"], CFG["G"], seed=0, b=0, h=0)
    idx, _ = O.build_index(u["K"], u["V"], CFG["C"], 1, seed=0, unit=0)
    O.decode_unit(u["q"], idx, args.p)
    ts, t_start = [], time.perf_counter()
    while time.perf_counter() - t_start < budget_s or len(ts) < 3:
        t0 = time.perf_counter()
        O.decode_unit(u["q"], idx, args.p)
        ts.append(time.perf_counter() - t0)
        if len(ts) >= 400:
            break
    val = float(np.mean(ts)) * CFG["B"] * CFG["Hkv"] * 1e6
    return {"value": val, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle",
            "sample": f"{len(ts)} oracle decode_unit calls on KV head 0 of C2 (n=131072, C=1024, G=4, p={args.p}; "
                      f"index from 1 untimed oracle Lloyd iteration), mean x 8 units = one layer-step"}


# ------------------------------------------------------------------ GPU arm
def _unit_bits(job):
    from synth import bf16_bits, make_unit
    seed, b, h, n, G = job
    u = make_unit(n, G, seed=seed, b=b, h=h)
    return seed, b, h, bf16_bits(u["K"]), bf16_bits(u["V"]), bf16_bits(u["q"])


def make_layers(seeds, dev, B=1, Hkv=None, n=None):
    """The synthetic layers (one per seed) as bf16 device tensors [B][Hkv][n][128],
    generated in parallel on the host cores (input generation only; synth/ holds no
    method arithmetic)."""
    import multiprocessing as mp

    import torch
    Hkv = Hkv or CFG["Hkv"]
    n = n or CFG["n"]
    G = CFG["G"]
    bf = lambda a: torch.from_numpy(a.view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    layers = {sd: {"K": torch.empty((B, Hkv, n, 128), dtype=torch.bfloat16, device=dev),
                   "V": torch.empty((B, Hkv, n, 128), dtype=torch.bfloat16, device=dev),
                   "q": torch.empty((B, Hkv * G, 128), dtype=torch.bfloat16, device=dev)} for sd in seeds}
    jobs = [(sd, b, h, n, G) for sd in seeds for b in range(B) for h in range(Hkv)]
    workers = max(1, min(len(jobs), len(os.sched_getaffinity(0)) - 1, 32))
    with mp.get_context("fork").Pool(workers) as pool:
        for sd, b, h, kb, vb, qb in pool.imap_unordered(_unit_bits, jobs, chunksize=4):
            L = layers[sd]
            L["K"][b, h] = bf(kb)
            L["V"][b, h] = bf(vb)
            L["q"][b, h * G:(h + 1) * G] = bf(qb)
    return [layers[sd] for sd in seeds]


C3 = dict(B=64, Hkv=8, n=32768, C=256, iters=10)


def measure_c3(T, dev, p, steps, timed_loop):
    """BASELINE.json configs[2] on this GPU: Llama-3-8B layer, 32K context, batch 64
    (512 units, 256 clusters each): decode layer-step vs the own dense decode (the global
    token split of the attention kernel: more units than half the CTAs)."""
    import torch
    L = make_layers([9000], dev, B=C3["B"], Hkv=C3["Hkv"], n=C3["n"])[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx = T.build_index(L["K"], L["V"], C3["C"], C3["iters"], group_size=CFG["G"], seed=9000)
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1)
    ex = idx.export()
    units = idx.units
    sizes = np.stack([np.bincount(ex["assign"][u], minlength=C3["C"]) for u in range(units)])
    out = torch.empty_like(L["q"])
    T.decode(L["q"], idx, p, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        T.decode(L["q"], idx, p, out=out)
    dout = torch.empty_like(L["q"])
    T.dense_decode(L["q"], L["K"], L["V"], out=dout)
    gd = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gd):
        T.dense_decode(L["q"], L["K"], L["V"], out=dout)
    k = max(10, min(steps, 50))
    timed_loop([g.replay], 3)
    ev = timed_loop([g.replay], k)
    torch.cuda.synchronize()
    us = 1e3 * float(np.mean([a.elapsed_time(b) for a, b in ev]))
    timed_loop([gd.replay], 3)
    ev = timed_loop([gd.replay], k)
    torch.cuda.synchronize()
    dus = 1e3 * float(np.mean([a.elapsed_time(b) for a, b in ev]))
    dbg = T.decode_debug(L["q"], idx, p)
    uf = sum(int(sizes[u][dbg["union_mask"][u].astype(bool)].sum()) for u in range(units)) / (units * C3["n"])
    dense_bytes = 2 * units * C3["n"] * 256
    res = {"workload": "C3: Llama-3-8B layer, 32K context, batch 64 (512 units), 256 clusters/KV head, "
                       f"p={p}, 1 GPU", "us_per_layer_step": us, "dense_us_per_layer_step": dus,
           "speedup_vs_dense": dus / us, "union_frac": uf, "dense_gbs": dense_bytes / (dus * 1e-6) / 1e9,
           "build_ms": build_ms}
    del L, idx
    torch.cuda.empty_cache()
    return res


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2502_12216_b200 import build as B
    B.build()
    from paper_2502_12216_b200 import tactic as T
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    T.device_check()
    G, n, C = CFG["G"], CFG["n"], CFG["C"]
    layers = make_layers([LAYERS * rank + l for l in range(LAYERS)], dev)

    # ---- index build per layer (tcgen05 k-means + relayout), timed separately
    T.build_index(layers[0]["K"][:, :1, :8192].contiguous(), layers[0]["V"][:, :1, :8192].contiguous(), 64, 2,
                  group_size=G)  # warm
    torch.cuda.synchronize()
    build_ms, iters_run = [], []
    for li, L in enumerate(layers):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L["index"] = T.build_index(L["K"], L["V"], C, CFG["iters"], group_size=G, seed=LAYERS * rank + li)
        e1.record()
        torch.cuda.synchronize()
        build_ms.append(e0.elapsed_time(e1))
        ex = L["index"].export()
        iters_run += ex["iters_run"].tolist()
        L["sizes"] = np.stack([np.bincount(ex["assign"][u], minlength=C) for u in range(L["index"].units)])
        L["out"] = torch.empty_like(L["q"])
    units = layers[0]["index"].units
    alg_tflop = 2.0 * n * C * 128 * sum(iters_run) / 1e12 / len(layers)   # per layer

    # cold L2 before every timed step: write a 256 MiB buffer (> 126 MB L2), then read a
    # second one so the dirty lines of the write are written back before the step starts
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_r = torch.ones(32 << 20, dtype=torch.int64, device=dev)
    flush_acc = torch.empty((), dtype=torch.int64, device=dev)

    def l2_flush():
        flush.fill_(1)
        torch.sum(flush_r, dim=0, out=flush_acc)

    # ---- one CUDA graph per layer: one decode layer-step
    for L in layers:
        T.decode(L["q"], L["index"], args.p, out=L["out"])
        torch.cuda.synchronize()
        L["graph"] = torch.cuda.CUDAGraph()
        with torch.cuda.graph(L["graph"]):
            T.decode(L["q"], L["index"], args.p, out=L["out"])
    torch.cuda.synchronize()

    def timed_loop(fns, steps, flush_each=True):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i, (a, b) in enumerate(evs):
            if flush_each:
                l2_flush()
            a.record()
            fns[i % len(fns)]()
            b.record()
        return evs

    # ---- one step = one decode step through all LAYERS synthetic layers, captured as ONE
    # CUDA graph (as a serving engine captures its decode step); every layer's decode starts
    # only after the previous layer's has completed (the entry kernel takes no programmatic
    # dependency), each layer reads its own K/V (512 MB per layer > L2) and L2 is flushed
    # before every step.  value = step time / LAYERS.
    def model_graph(fn):
        for L in layers:
            fn(L)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for L in layers:
                fn(L)
        torch.cuda.synchronize()
        return g

    def per_layer_us(evs):
        return 1e3 * float(np.mean([a.elapsed_time(b) for a, b in evs])) / len(layers)

    gmodel = model_graph(lambda L: T.decode(L["q"], L["index"], args.p, out=L["out"]))
    timed_loop([gmodel.replay], args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        evs = timed_loop([gmodel.replay], args.steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # keep the GPU busy a little longer for the clock sampler (not part of the number)
        timed_loop([gmodel.replay], min(args.steps, 100))
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms)) / len(layers)   # per layer-step
    ms_model_step = float(np.mean(step_ms))

    # the same layer-step as its own graph (one graph launch per layer, as in r01)
    replays = [L["graph"].replay for L in layers]
    timed_loop(replays, 2 * LAYERS)
    torch.cuda.synchronize()
    iso_ev = timed_loop(replays, max(4 * LAYERS, min(args.steps, 200)))
    torch.cuda.synchronize()
    iso_us = 1e3 * float(np.mean([a.elapsed_time(b) for a, b in iso_ev]))
    if world > 1:
        t = torch.tensor([ms_model_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_model_step = float(t.item())
        ms = ms_model_step / len(layers)

    # ---- per-stage breakdown (selection / attention / merge), events between stages
    st = []
    for i in range(max(3 * LAYERS, min(args.steps, 200))):
        L = layers[i % len(layers)]
        l2_flush()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        T.decode_profiled(L["q"], L["index"], args.p, ev, out=L["out"])
        st.append(ev)
    torch.cuda.synchronize()
    sel_us = 1e3 * float(np.mean([e[0].elapsed_time(e[1]) for e in st]))
    att_us = 1e3 * float(np.mean([e[1].elapsed_time(e[2]) for e in st]))
    mrg_us = 1e3 * float(np.mean([e[2].elapsed_time(e[3]) for e in st]))

    # ---- the attention kernel's launch duration for the roofline: S8 + S9 alone over each
    # layer's work list (left by the decodes above), the 8 layers' launches back to back in
    # one graph (8 distinct unions, together larger than L2), cold L2 before each replay
    for L in layers:
        T.decode(L["q"], L["index"], args.p, out=L["out"])
    gatt = model_graph(lambda L: T.decode_attention_only(L["q"], L["index"], L["out"]))
    timed_loop([gatt.replay], 3)
    torch.cuda.synchronize()
    att_ev = timed_loop([gatt.replay], max(10, min(args.steps, 50)))
    torch.cuda.synchronize()
    att_launch_us = per_layer_us(att_ev)

    # ---- algorithmic bytes from the selections the GPU made (mean over layers)
    bms = []
    for L in layers:
        dbg = T.decode_debug(L["q"], L["index"], args.p)
        assert torch.equal(dbg["out"], L["out"]), "debug decode must reproduce the graph output"
        bms.append(step_bytes(dbg, L["sizes"], G, n, C))
    bm = {k: float(np.mean([b[k] for b in bms])) for k in bms[0]}
    bm["union_frac_per_layer"] = [round(b["union_frac"], 5) for b in bms]

    # ---- dense baseline (own split-KV flash-decode over the caller's K/V), same layers
    dgraphs = []
    for L in layers:
        L["dout"] = torch.empty_like(L["q"])
        T.dense_decode(L["q"], L["K"], L["V"], out=L["dout"])
        gd = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gd):
            T.dense_decode(L["q"], L["K"], L["V"], out=L["dout"])
        dgraphs.append(gd.replay)
    timed_loop(dgraphs, 3 * LAYERS)
    torch.cuda.synchronize()
    devs = timed_loop(dgraphs, max(2 * LAYERS, min(args.steps, 100)))
    torch.cuda.synchronize()
    dense_iso_ms = float(np.mean([a.elapsed_time(b) for a, b in devs]))
    gdm = model_graph(lambda L: T.dense_decode(L["q"], L["K"], L["V"], out=L["dout"]))
    timed_loop([gdm.replay], 3)
    torch.cuda.synchronize()
    dev_m = timed_loop([gdm.replay], max(10, min(args.steps, 50)))
    torch.cuda.synchronize()
    dense_ms = per_layer_us(dev_m) * 1e-3
    dense_bytes = 2 * units * n * 128 * 2 + 2 * units * G * 128 * 2

    # ---- e2e through the C ABI with host buffers (H2D q, D2H out inside the timed region)
    for L in layers:
        L["q_host"] = L["q"].cpu().pin_memory()
        L["o_host"] = torch.empty_like(L["q_host"]).pin_memory()
        T.decode_host(L["q_host"], L["index"], args.p, L["o_host"])
    e2e = []
    for i in range(max(2 * LAYERS, min(args.steps, 200))):
        L = layers[i % len(layers)]
        l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        T.decode_host(L["q_host"], L["index"], args.p, L["o_host"])
        b.record()
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_ms = float(np.mean(e2e))
    if world > 1:
        t = torch.tensor([e2e_ms, dense_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms, dense_ms = float(t[0]), float(t[1])
    qd = layers[0]["q"]
    index = layers[0]["index"]
    build_ms = float(np.mean(build_ms))
    c3 = measure_c3(T, dev, args.p, args.steps, timed_loop) if (args.c3 and world == 1) else None

    # ---- C4 (BASELINE.json configs[3]: 1M tokens sequence-sharded over 8 GPUs): on this
    # single GPU, one shard's compute per decode step (a C2-shaped shard: 131072 tokens x
    # 8 KV heads, C = 1024) through the three sharded stages + the final LSE merge, with the
    # three collectives (MAX all-reduce, SUM all-reduce, all-gather) absent (world size 1)
    c4 = None
    if args.c4 and world == 1:
        L = layers[0]
        lm = torch.empty((units, G, 2), dtype=torch.float64, device=dev)
        ms_ = torch.empty((units, G, 1 + T.SHARD_GRID_T), dtype=torch.float64, device=dev)
        op = torch.empty((units, G, 128), dtype=torch.float32, device=dev)
        lp = torch.empty((units, G), dtype=torch.float32, device=dev)
        mo = torch.empty((units * G, 128), dtype=torch.bfloat16, device=dev)

        def shard_step():
            T.decode_stage1(L["q"], L["index"], lm)
            T.decode_stage1b(L["index"], lm, ms_)
            T.decode_stage2(L["q"], L["index"], args.p, lm, ms_, op, lp)
            T.lse_merge(op.view(1, units * G, 128), lp.view(1, units * G), out=mo)

        shard_step()
        gs = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gs):
            shard_step()
        timed_loop([gs.replay], 5)
        torch.cuda.synchronize()
        ev = timed_loop([gs.replay], max(20, min(args.steps, 100)))
        torch.cuda.synchronize()
        c4 = {"workload": "C4 shard: 131072 tokens x 8 KV heads (one of 8 shards of a 1M-token context), C = 1024, "
                          f"p={args.p}; stage1 + stage1b + stage2 + LSE merge on 1 GPU, collectives not included",
              "us_per_shard_step": 1e3 * float(np.mean([a.elapsed_time(b) for a, b in ev])),
              "dense_us_per_shard_step": dense_ms * 1e3}

    # ---- Table-1 diagnostics (NEXT 3) over the same layers: Optimal /
    # Cluster-Optimal / Tactic budgets, achieved cumulative score and success rate
    table1 = None
    if args.table1 and world == 1:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from table1 import public, table1_stats
        acc = {}
        for L in layers:
            st = public(table1_stats(T, L["q"], L["index"], L["sizes"], (0.5, 0.9)))
            for pk, d in st.items():
                for k, v in d.items():
                    acc.setdefault(pk, {}).setdefault(k, []).append(v)
        table1 = {pk: {k: (float(np.sum(v)) if k == "instances" else float(np.mean(v))) for k, v in d.items()}
                  for pk, d in acc.items()}
        # Fig. 5: threshold rule vs a fixed budget of the same mean size (first layer)
        from table1 import fig5_variance
        table1["fig5_variance_layer0"] = fig5_variance(T, layers[0]["q"], layers[0]["index"], layers[0]["sizes"],
                                                       layers[0]["K"], layers[0]["V"], args.p)

    # ---- GQA union vs per-head loading (NEXT 2: union up to 1.65x faster)
    ablation = None
    if args.ablation and world == 1:
        own_tok, uni_tok = [], []
        for L in layers:
            L["o_ph"] = torch.empty_like(L["q"])
        gph = model_graph(lambda L: T.decode_per_head(L["q"], L["index"], args.p, out=L["o_ph"]))
        for L in layers:
            dbg = T.decode_debug(L["q"], L["index"], args.p)
            for u in range(units):
                uni_tok.append(int(L["sizes"][u][dbg["union_mask"][u].astype(bool)].sum()))
                own_tok.append(sum(int(L["sizes"][u][dbg["order"][u, g][:dbg["J"][u, g]]].sum()) for g in range(G)))
        timed_loop([gph.replay], 3)
        torch.cuda.synchronize()
        ev = timed_loop([gph.replay], max(10, min(args.steps, 50)))
        torch.cuda.synchronize()
        ph_us = per_layer_us(ev)
        ablation = {"per_head_us_per_layer_step": ph_us, "union_us_per_layer_step": ms * 1e3,
                    "union_speedup": ph_us / (ms * 1e3),
                    "kv_tokens_per_head_loading": float(np.sum(own_tok)) / len(layers),
                    "kv_tokens_union": float(np.sum(uni_tok)) / len(layers),
                    "paper": "union up to 1.65x faster than per-head loading (P:695)"}

    # ---- target-fraction sweep (BASELINE.json configs[4], C5): same layers, graph per (p,
    # layer), device-timed like the headline, plus the union fraction the GPU selected
    sweep = []
    if args.sweep and world == 1:
        for p in (0.5, 0.8, 0.9, 0.95, 0.99, 1.0):
            for L in layers:
                L["o_sw"] = torch.empty_like(L["q"])
            gp = model_graph(lambda L: T.decode(L["q"], L["index"], p, out=L["o_sw"]))
            timed_loop([gp.replay], 3)
            torch.cuda.synchronize()
            ev = timed_loop([gp.replay], max(10, min(args.steps, 50)))
            torch.cuda.synchronize()
            us = per_layer_us(ev)
            del gp
            uf = []
            for L in layers:
                if p >= 1.0:
                    uf.append(float((L["sizes"] > 0).sum() and 1.0))
                else:
                    dbg = T.decode_debug(L["q"], L["index"], p)
                    uf.append(sum(int(L["sizes"][u][dbg["union_mask"][u].astype(bool)].sum())
                                  for u in range(units)) / (units * n))
            sweep.append({"p": p, "us_per_layer_step": us, "speedup_vs_dense": dense_ms * 1e3 / us,
                          "union_frac": float(np.mean(uf))})

    if rank != 0:
        return
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING)"
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    attn_bytes = bm["union_kv"] + bm["q_out"] // 2 + (n_sm + index.units) * G * 129 * 4   # K/V, q, partials
    att_gbs = attn_bytes / (att_launch_us * 1e-6) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get("attention_kernel_sparse_bytes_per_launch")
    except Exception:
        pass
    value_us = ms * 1e3 / world
    line = {
        "metric": METRIC, "value": value_us, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_model_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": _config(args, world),
        # per decode step: score+rank, sample, fit, attention
        "gpu_launches": (1 if args.p >= 1 else 4) * LAYERS * args.steps,
        "roofline": {"bound": "hbm", "kernel": "attention_kernel<4,false> (S8 sparse split-KV)",
                     "achieved": att_gbs, "peak": hbm, "unit": "GB/s", "frac": att_gbs / hbm,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": attn_bytes, "us_per_launch": att_launch_us,
                     "timing": "S8+S9 alone, 8 layers' launches back to back in one graph (no PDL), cold L2 "
                               "per replay, CUDA events; mean per launch",
                     "us_per_launch_event_bracketed_in_step": att_us},
        "step_roofline": {"bytes_per_step": bm["total"], "achieved_gbs": bm["total"] / (ms * 1e-3) / 1e9,
                          "frac": bm["total"] / (ms * 1e-3) / 1e9 / hbm, "bytes": bm},
        "stages_us": {"selection_S1_S7": sel_us, "attention_S8": att_us, "merge_S9": mrg_us},
        "dense": {"us_per_layer_step": dense_ms * 1e3, "gbs": dense_bytes / (dense_ms * 1e-3) / 1e9,
                  "frac": dense_bytes / (dense_ms * 1e-3) / 1e9 / hbm, "bytes": dense_bytes},
        "speedup_vs_dense": dense_ms / ms,
        "isolated_layer_graph": {"us_per_layer_step": iso_us, "dense_us_per_layer_step": dense_iso_ms * 1e3,
                                 "speedup_vs_dense": dense_iso_ms * 1e3 / iso_us,
                                 "what": "each layer-step as its own CUDA graph, L2 flushed before each (includes one graph launch per layer)"},
        "p_sweep": sweep or None,
        "c3": c3,
        "c4_shard": c4,
        "table1": table1,
        "gqa_union_ablation": ablation,
        "build": {"ms": build_ms, "iters_run": iters_run, "alg_tflop": alg_tflop,
                  "alg_tflops": alg_tflop / (build_ms * 1e-3),
                  "exec_tflops_split_bf16": 2 * alg_tflop / (build_ms * 1e-3)},
        "e2e": {"value": e2e_ms * 1e3 / world, "unit": UNIT, "h2d_bytes_per_step": int(qd.numel() * 2),
                "d2h_bytes_per_step": int(qd.numel() * 2)},
        "clocks": clk.summary(),
        "context": PAPER_CONTEXT,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=float, default=0.9)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", type=int, default=1, help="1: add the C5 target-fraction sweep (p_sweep)")
    ap.add_argument("--c3", type=int, default=1, help="1: add the C3 batch-64 32K measurement (configs[2])")
    ap.add_argument("--table1", type=int, default=1, help="1: add the Table-1 diagnostics (budgets, success)")
    ap.add_argument("--c4", type=int, default=1, help="1: add the C4 per-shard sequence-sharded measurement")
    ap.add_argument("--ablation", type=int, default=1, help="1: add the GQA union vs per-head loading ablation")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
