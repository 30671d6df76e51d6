#!/usr/bin/env python
"""bench.py -- Tactic decode-attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--p 0.9]

A *step* is one decode layer-step of the whole hot path (S1-S9: centroid scoring, cluster
sort, sampled exact scoring, a/x+b fit, estimated-mass selection, GQA union + work list,
split-KV flash-decode, LSE merge) over one C2 layer: Llama-3-8B shape (32 Q / 8 KV
heads, d=128), 128K context, batch 1, 1024 clusters per KV head, p=0.9, bf16 KV.
The index (tcgen05 k-means + cluster-contiguous relayout) is built once per layer and
timed separately ("build").  N GPUs (`--gpus N` re-launches itself under torchrun, one
rank per GPU): the 8 units (KV heads) of every C2 layer are split into contiguous blocks,
one per rank (batch x KV-head sharding; no collective on the data
path), each rank builds and decodes its block, and the reported time is the max over
ranks of the layer-step time -- the same job on more GPUs ("scaling": "strong").  C3 (batch
64 x 32K, 512 units) is sharded the same way (512 / N units per GPU) and reported in `c3`;
C4 (sequence-sharded, one 131072-token shard per GPU) is timed with its three NCCL
collectives in `c4`.

Layers: the timed steps cycle over LAYERS = 8 distinct synthetic layers (seeds 0..7),
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
    return {"workload": f"{WORKLOAD}: Llama-3-8B layer (32 Q / 8 KV heads, d=128), 128K context, batch 1, "
                        f"1024 clusters/KV head, p={args.p}",
            "global_batch": 1, "seq_len": CFG["n"], "n_clusters": CFG["C"], "p": args.p,
            "parallelism": f"batch x KV-head: the layer's 8 units in contiguous blocks over {n_gpus} GPU(s) "
                           f"(units per GPU: {[b - a for a, b in (_unit_block(8, n_gpus, r) for r in range(n_gpus))]}), "
                           "no data-path collective; time = max over ranks",
            "l2": "cold L2 before every timed step: 256 MiB buffer written, then a 256 MiB buffer read (write-back drained); "
                  "within a step each layer reads its own K/V (512 MB per layer > L2)",
            "step": f"one decode step through all {LAYERS} synthetic layers, one CUDA graph, layers serialised "
                    f"(no cross-layer overlap); value = step time / {LAYERS}",
            "inputs": f"tactic-synth-v1 (synth/), {LAYERS} layers (seeds 0..{LAYERS - 1}), unit (b, h) seeded by (seed, b, h)"}


def _unit_block(units, world, rank):
    from paper_2502_12216_b200.sharded import unit_block
    return unit_block(units, world, rank)


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
def step_bytes(dbg, sizes, G, n, C, sc):
    """Algorithmic bytes of one layer-step: fp32 centroids, sampled K rows not re-read by the
    attention, selected (union) K+V rows, q/out, from the selection the GPU actually made
    (sc: the index's sampling constants, tactic_index_sample_constants)."""
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
    idx, _ = O.build_index(u["K"], u["V"], CFG["C"], CFG["iters"], seed=0, unit=0)   # setup, untimed
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
                             "sample": f"1 of 8 units per step (KV head 0 of layer 0, n=131072, C=1024; index from "
                                       f"the oracle's own {CFG['iters']}-iteration k-means, untimed), scaled x8 to a layer-step"},
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


def cpu_baseline(args, K, V, q, cents, assign, budget_s=12.0):
    """Time the oracle decode (as it stands) on a bounded sample of the C2 workload: unit 0
    of layer 0 on the SAME clustering the GPU decodes (the GPU's 10-iteration index,
    exported), so both sides select from one index."""
    from oracle import tactic_oracle as O
    idx = O.make_index(K, V, cents, assign)
    O.decode_unit(q, idx, args.p)
    ts, t_start = [], time.perf_counter()
    while time.perf_counter() - t_start < budget_s or len(ts) < 3:
        t0 = time.perf_counter()
        O.decode_unit(q, idx, args.p)
        ts.append(time.perf_counter() - t0)
        if len(ts) >= 400:
            break
    val = float(np.mean(ts)) * CFG["B"] * CFG["Hkv"] * 1e6
    return {"value": val, "unit": UNIT, "cores": _cpu_threads(), "kind": "oracle",
            "sample": f"{len(ts)} oracle decode_unit calls on KV head 0 of C2 layer 0 (n=131072, C=1024, G=4, "
                      f"p={args.p}; the GPU's {CFG['iters']}-iteration clustering, exported), mean x 8 units = one "
                      "layer-step"}


# ------------------------------------------------------------------ GPU arm
def _unit_bits(job):
    from synth import bf16_bits, make_unit
    key, j, seed, b, h, n, G, q_seed = job
    u = make_unit(n, G, seed=seed, b=b, h=h)
    qb = bf16_bits(u["q"])
    if q_seed is not None:   # sequence-sharded C4: every shard sees the query of shard 0
        qb = bf16_bits(make_unit(n, G, seed=q_seed, b=b, h=h)["q"])
    return key, j, bf16_bits(u["K"]), bf16_bits(u["V"]), qb


def make_layers(seeds, dev, pairs, n=None, q_seed=None):
    """One synthetic layer per seed holding the units `pairs` = [(b, h), ...] (this rank's
    block), as bf16 device tensors K, V [1][len(pairs)][n][128] and q [1][len(pairs) G][128];
    unit (b, h) of layer `seed` is make_unit(seed, b, h) whichever rank holds it.  Generated
    in parallel on the host cores (input generation only; synth/ holds no method arithmetic)."""
    import multiprocessing as mp

    import torch
    n = n or CFG["n"]
    G = CFG["G"]
    U = len(pairs)
    bf = lambda a: torch.from_numpy(a.view(np.int16)).to(dev).view(torch.bfloat16)  # noqa: E731
    layers = {sd: {"K": torch.empty((1, U, n, 128), dtype=torch.bfloat16, device=dev),
                   "V": torch.empty((1, U, n, 128), dtype=torch.bfloat16, device=dev),
                   "q": torch.empty((1, U * G, 128), dtype=torch.bfloat16, device=dev), "seed": sd,
                   "pairs": list(pairs)} for sd in seeds}
    jobs = [(sd, j, sd, b, h, n, G, q_seed) for sd in seeds for j, (b, h) in enumerate(pairs)]
    workers = max(1, min(len(jobs), len(os.sched_getaffinity(0)) - 1, 32))
    with mp.get_context("fork").Pool(workers) as pool:
        for sd, j, kb, vb, qb in pool.imap_unordered(_unit_bits, jobs, chunksize=2):
            L = layers[sd]
            L["K"][0, j] = bf(kb)
            L["V"][0, j] = bf(vb)
            L["q"][0, j * G:(j + 1) * G] = bf(qb)
    return [layers[sd] for sd in seeds]


C3 = dict(B=64, Hkv=8, n=32768, C=256, iters=10, seed=9000)
C4 = dict(n_shard=131072, Hkv=8, C=1024, iters=10, seed=7000)


class Timer:
    """CUDA-event timing on the launching stream with an L2 flush before every timed
    replay, barriers around the timed region and the max over ranks."""

    def __init__(self, dev, world):
        import torch
        self.world = world
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.flush_r = torch.ones(32 << 20, dtype=torch.int64, device=dev)
        self.flush_acc = torch.empty((), dtype=torch.int64, device=dev)
        self.dev = dev

    def l2_flush(self):
        # cold L2 before every timed step: write a 256 MiB buffer (> 126 MB L2), then read a
        # second one so the dirty lines of the write are written back before the step starts
        import torch
        self.flush.fill_(1)
        torch.sum(self.flush_r, dim=0, out=self.flush_acc)

    def loop(self, fns, steps, flush_each=True):
        import torch
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i, (a, b) in enumerate(evs):
            if flush_each:
                self.l2_flush()
            a.record()
            fns[i % len(fns)]()
            b.record()
        return evs

    def barrier(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, *vals):
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return vals if len(vals) > 1 else vals[0]
        t = torch.tensor(list(vals), dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out = [float(x) for x in t.tolist()]
        return out if len(out) > 1 else out[0]

    def timed(self, fns, steps, warmup=3):
        """mean ms per call over `steps` timed calls; max over ranks"""
        import torch
        self.loop(fns, warmup)
        self.barrier()
        evs = self.loop(fns, steps)
        torch.cuda.synchronize()
        ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
        self.barrier()
        return self.max_over_ranks(ms)


def capture(fn):
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g


def phase_timeline(T, L, args, tm, reps=20):
    """In-graph %globaltimer phases of one decode layer-step (S1-S3 score + rank, S4 sample,
    S5-S7 fit + union work list, S8-S9 attention + merge) on layer L, from an index built
    with the library's debug timeline (TACTIC_TLOG=1: each decode kernel stamps its first
    CTA's start and the last CTA's end).  Medians over `reps` cold-L2 replays."""
    import torch
    os.environ["TACTIC_TLOG"] = "1"
    try:
        idx = T.build_index(L["K"], L["V"], CFG["C"], CFG["iters"], group_size=CFG["G"], seed=L["seed"],
                            unit_offset=L["u0"])
    finally:
        del os.environ["TACTIC_TLOG"]
    out = torch.empty_like(L["q"])
    g = capture(lambda: T.decode(L["q"], idx, args.p, out=out))
    rows = []
    for _ in range(reps):
        tm.l2_flush()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        tl = idx.debug_timing().astype(np.int64)[1536:1536 + 20].reshape(5, 4)
        k_rank, k_sample, k_fit, k_att = 1, 2, 3, 4
        t0 = tl[k_rank, 0]
        rows.append([(tl[k_rank, 2] - t0), (tl[k_sample, 2] - tl[k_rank, 2]), (tl[k_fit, 2] - tl[k_sample, 2]),
                     (tl[k_att, 2] - tl[k_fit, 2]), (tl[k_att, 2] - t0)])
    med = np.median(np.array(rows, dtype=np.float64), axis=0) / 1e3
    del g, idx
    return {"S1_S3_score_rank": med[0], "S4_sample": med[1], "S5_S7_fit_union": med[2],
            "S8_S9_attention_merge": med[3], "total": med[4],
            "method": "in-graph %globaltimer (TACTIC_TLOG=1 index of layer 0): score_rank start -> its last CTA "
                      "end -> sample end -> fit end -> attention end; S9 is fused into the attention kernel; "
                      f"median of {reps} cold-L2 replays; debug stamps add ~0.5 us"}


def measure_c3(T, dev, args, rank, world, tm):
    """BASELINE.json configs[2]: Llama-3-8B layer, 32K context, batch 64 (512 units, 256
    clusters each), the 512 units sharded over the ranks in contiguous blocks: decode
    layer-step vs the own dense decode, max over ranks."""
    import torch
    from paper_2502_12216_b200.sharded import block_units, unit_block
    units = C3["B"] * C3["Hkv"]
    u0, u1 = unit_block(units, world, rank)
    L = make_layers([C3["seed"]], dev, block_units(units, C3["Hkv"], world, rank), n=C3["n"])[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx = T.build_index(L["K"], L["V"], C3["C"], C3["iters"], group_size=CFG["G"], seed=C3["seed"], unit_offset=u0)
    e1.record()
    torch.cuda.synchronize()
    build_ms = e0.elapsed_time(e1)
    ex = idx.export()
    sizes = np.stack([np.bincount(ex["assign"][u], minlength=C3["C"]) for u in range(idx.units)])
    out = torch.empty_like(L["q"])
    g = capture(lambda: T.decode(L["q"], idx, args.p, out=out))
    dout = torch.empty_like(L["q"])
    gd = capture(lambda: T.dense_decode(L["q"], L["K"], L["V"], out=dout))
    k = max(10, min(args.steps, 50))
    us = 1e3 * tm.timed([g.replay], k)
    dus = 1e3 * tm.timed([gd.replay], k)
    dbg = T.decode_debug(L["q"], idx, args.p)
    tok = sum(int(sizes[u][dbg["union_mask"][u].astype(bool)].sum()) for u in range(idx.units))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(tok)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        tok = float(t.item())
    uf = tok / (units * C3["n"])
    dense_bytes = 2 * units * C3["n"] * 256
    res = {"workload": f"C3: Llama-3-8B layer, 32K context, batch 64 (512 units), 256 clusters/KV head, p={args.p}; "
                       f"units sharded over {world} GPU(s) ({u1 - u0} on rank {rank}), time = max over ranks",
           "us_per_layer_step": us, "dense_us_per_layer_step": dus, "speedup_vs_dense": dus / us,
           "union_frac": uf, "dense_gbs_job": dense_bytes / (dus * 1e-6) / 1e9, "build_ms": build_ms,
           "units_per_gpu": u1 - u0, "n_gpus": world,
           "gpu_launches_per_step": 5}   # score (all heads), rank, sample, fit, attention
    del L, idx, g, gd
    torch.cuda.empty_cache()
    return res


def measure_c4(T, dev, args, rank, world, tm):
    """BASELINE.json configs[3] scaled to the job's GPUs: a context of world x 131072 tokens
    sequence-sharded one shard per rank (8 KV heads per shard, C = 1024; world = 8 is the 1M
    configuration).  One decode step = stage1 -> NCCL all-reduce MAX -> stage1b -> NCCL
    all-reduce SUM -> stage2 -> NCCL all-gather of (o, lse) -> LSE merge (reading 23),
    timed as one step, plus the compute alone and the three collectives alone."""
    import torch
    import torch.distributed as dist
    G, Hkv, n = CFG["G"], C4["Hkv"], C4["n_shard"]
    pairs = [(0, h) for h in range(Hkv)]
    L = make_layers([C4["seed"] + rank], dev, pairs, n=n, q_seed=C4["seed"] if rank else None)[0]
    idx = T.build_index(L["K"], L["V"], C4["C"], C4["iters"], group_size=G, seed=C4["seed"] + rank)
    units = Hkv
    q = L["q"]
    lm = torch.empty((units, G, 2), dtype=torch.float64, device=dev)
    ms_ = torch.empty((units, G, 1 + T.SHARD_GRID_T), dtype=torch.float64, device=dev)
    op = torch.empty((units, G, 128), dtype=torch.float32, device=dev)
    lp = torch.empty((units, G), dtype=torch.float32, device=dev)
    o_all = torch.empty((world, units * G, 128), dtype=torch.float32, device=dev)
    l_all = torch.empty((world, units * G), dtype=torch.float32, device=dev)
    out = torch.empty((units * G, 128), dtype=torch.bfloat16, device=dev)

    def compute_only():
        T.decode_stage1(q, idx, lm)
        T.decode_stage1b(idx, lm, ms_)
        T.decode_stage2(q, idx, args.p, lm, ms_, op, lp)
        T.lse_merge(op.view(1, units * G, 128), lp.view(1, units * G), out=out)

    def collectives_only():
        dist.all_reduce(lm, op=dist.ReduceOp.MAX)
        dist.all_reduce(ms_, op=dist.ReduceOp.SUM)
        dist.all_gather_into_tensor(o_all, op.view(units * G, 128))
        dist.all_gather_into_tensor(l_all, lp.view(units * G))

    def step():
        T.decode_stage1(q, idx, lm)
        dist.all_reduce(lm, op=dist.ReduceOp.MAX)
        T.decode_stage1b(idx, lm, ms_)
        dist.all_reduce(ms_, op=dist.ReduceOp.SUM)
        T.decode_stage2(q, idx, args.p, lm, ms_, op, lp)
        dist.all_gather_into_tensor(o_all, op.view(units * G, 128))
        dist.all_gather_into_tensor(l_all, lp.view(units * G))
        T.lse_merge(o_all, l_all, out=out)

    k = max(20, min(args.steps, 100))
    how = "one CUDA graph per step (NCCL collectives captured)"
    try:
        step()
        tm.barrier()
        gs = capture(step)
        step_fn = gs.replay
    except Exception as e:  # noqa: BLE001  (capture of the collectives unsupported: eager)
        torch.cuda.synchronize()
        how = f"eager launches (graph capture failed: {type(e).__name__})"
        step_fn = step
    step_us = 1e3 * tm.timed([step_fn], k)
    gc = capture(compute_only)
    comp_us = 1e3 * tm.timed([gc.replay], k)
    coll_us = 1e3 * tm.timed([collectives_only], k)
    res = {"workload": f"C4: {world} x 131072-token context (1M at 8 GPUs) sequence-sharded, one shard (8 KV heads, "
                       f"C = 1024) per GPU, p={args.p}; stage1 -> all_reduce MAX -> stage1b -> all_reduce SUM -> "
                       "stage2 -> all_gather (o, lse) -> LSE merge",
           "us_per_step": step_us, "compute_only_us": comp_us, "collectives_only_us": coll_us,
           "timing": how + "; collectives alone: eager NCCL calls on the same buffers", "n_gpus": world,
           "collective_bytes": {"all_reduce_max": lm.numel() * 8, "all_reduce_sum": ms_.numel() * 8,
                                "all_gather": (o_all.numel() + l_all.numel()) * 4}}
    del L, idx
    torch.cuda.empty_cache()
    return res


def run_gpu(args, rank, world, local_rank):
    import torch
    from paper_2502_12216_b200 import build as B
    from paper_2502_12216_b200.sharded import block_units, unit_block
    B.build()
    from paper_2502_12216_b200 import tactic as T
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    T.device_check()
    G, n, C = CFG["G"], CFG["n"], CFG["C"]
    units_job = CFG["B"] * CFG["Hkv"]
    u0, u1 = unit_block(units_job, world, rank)
    pairs = block_units(units_job, CFG["Hkv"], world, rank)
    layers = make_layers(list(range(LAYERS)), dev, pairs)
    tm = Timer(dev, world)

    # ---- index build per layer (tcgen05 k-means + relayout), timed separately
    T.build_index(layers[0]["K"][:, :1, :8192].contiguous(), layers[0]["V"][:, :1, :8192].contiguous(), 64, 2,
                  group_size=G)  # warm
    torch.cuda.synchronize()
    build_ms, build_gpu_ms, iters_run = [], [], []
    for L in layers:
        L["u0"] = u0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L["index"] = T.build_index(L["K"], L["V"], C, CFG["iters"], group_size=G, seed=L["seed"], unit_offset=u0)
        e1.record()
        torch.cuda.synchronize()
        build_ms.append(e0.elapsed_time(e1))
        build_gpu_ms.append(L["index"].info()["build_gpu_ms"])
        ex = L["index"].export()
        iters_run += ex["iters_run"].tolist()
        L["sizes"] = np.stack([np.bincount(ex["assign"][u], minlength=C) for u in range(L["index"].units)])
        L["out"] = torch.empty_like(L["q"])
        if L["seed"] == 0:
            L["export"] = ex
    units = layers[0]["index"].units
    sc = layers[0]["index"].sample_constants()
    alg_tflop = 2.0 * n * C * 128 * sum(iters_run) / 1e12 / len(layers)   # per layer (this rank's units)

    def model_graph(fn):
        return capture(lambda: [fn(L) for L in layers])

    # ---- one step = one decode step through all LAYERS synthetic layers, captured as ONE
    # CUDA graph (as a serving engine captures its decode step); every layer's decode starts
    # only after the previous layer's has completed (the entry kernel takes no programmatic
    # dependency), each layer reads its own K/V (512 MB per layer > L2) and L2 is flushed
    # before every step.  value = max over ranks of the step time / LAYERS.
    gmodel = model_graph(lambda L: T.decode(L["q"], L["index"], args.p, out=L["out"]))
    tm.loop([gmodel.replay], args.warmup)
    tm.barrier()
    with ClockSampler(local_rank) as clk:
        evs = tm.loop([gmodel.replay], args.steps)
        torch.cuda.synchronize()
        tm.barrier()
        # keep the GPU busy a little longer for the clock sampler (not part of the number)
        tm.loop([gmodel.replay], min(args.steps, 100))
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms_model_step = tm.max_over_ranks(float(np.mean(step_ms)))
    ms = ms_model_step / len(layers)   # per layer-step (job: max over ranks)
    step_p50 = float(np.median(step_ms)) / len(layers)
    step_p99 = float(np.percentile(step_ms, 99)) / len(layers)

    # ---- in-graph phase timeline (S1-S3 / S4 / S5-S7 / S8-S9) of layer 0
    phases = phase_timeline(T, layers[0], args, tm)

    # ---- the same layer-step as its own graph (one graph launch per layer, as in r01)
    for L in layers:
        L["graph"] = capture(lambda L=L: T.decode(L["q"], L["index"], args.p, out=L["out"]))
    iso_us = 1e3 * tm.timed([L["graph"].replay for L in layers], max(4 * LAYERS, min(args.steps, 200)), 2 * LAYERS)

    # ---- the attention kernel's launch duration for the roofline: S8 + S9 alone over each
    # layer's work list (left by the decodes above), the 8 layers' launches back to back in
    # one graph (8 distinct unions, together larger than L2), cold L2 before each replay
    for L in layers:
        T.decode(L["q"], L["index"], args.p, out=L["out"])
    gatt = model_graph(lambda L: T.decode_attention_only(L["q"], L["index"], L["out"]))
    att_launch_us = 1e3 * tm.timed([gatt.replay], max(10, min(args.steps, 50))) / len(layers)

    # ---- algorithmic bytes from the selections the GPU made (mean over layers)
    bms = []
    for L in layers:
        dbg = T.decode_debug(L["q"], L["index"], args.p)
        assert same_decode(dbg["out"], L["out"]), "debug decode must reproduce the graph output"
        bms.append(step_bytes(dbg, L["sizes"], G, n, C, sc))
    bm = {k: float(np.mean([b[k] for b in bms])) for k in bms[0]}
    bm["union_frac_per_layer"] = [round(b["union_frac"], 5) for b in bms]

    # ---- dense baseline (own split-KV flash-decode over the caller's K/V), same layers
    for L in layers:
        L["dout"] = torch.empty_like(L["q"])
    dgraphs = [capture(lambda L=L: T.dense_decode(L["q"], L["K"], L["V"], out=L["dout"])).replay for L in layers]
    dense_iso_ms = tm.timed(dgraphs, max(2 * LAYERS, min(args.steps, 100)), 3 * LAYERS)
    gdm = model_graph(lambda L: T.dense_decode(L["q"], L["K"], L["V"], out=L["dout"]))
    dense_ms = tm.timed([gdm.replay], max(10, min(args.steps, 50))) / len(layers)
    dense_bytes = 2 * units_job * n * 128 * 2 + 2 * units_job * G * 128 * 2

    # ---- e2e through the C ABI with host buffers: tactic_decode_host (pinned q in, the
    # decode, out back, one synchronising call; the library replays its captured graph)
    for L in layers:
        L["q_host"] = L["q"].cpu().pin_memory()
        L["o_host"] = torch.empty_like(L["q_host"]).pin_memory()
        T.decode_host(L["q_host"], L["index"], args.p, L["o_host"])
        assert same_decode(L["o_host"], L["out"].cpu()), "host-buffer decode must reproduce the device decode"
    e2e = []
    tm.barrier()
    for i in range(max(2 * LAYERS, min(args.steps, 200))):
        L = layers[i % len(layers)]
        tm.l2_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        T.decode_host(L["q_host"], L["index"], args.p, L["o_host"])
        b.record()
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_ms = tm.max_over_ranks(float(np.mean(e2e)))
    build_ms = float(np.mean(build_ms))
    build_gpu_ms = float(np.mean(build_gpu_ms))

    c3 = measure_c3(T, dev, args, rank, world, tm) if args.c3 else None
    c4 = measure_c4(T, dev, args, rank, world, tm) if args.c4 else None
    if c4:  # like for like: one step per graph launch, cold L2 (C2's isolated layer-step)
        c4["compute_vs_c2_isolated_layer"] = c4["compute_only_us"] / iso_us

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
        ph_us = 1e3 * tm.timed([gph.replay], max(10, min(args.steps, 50))) / len(layers)
        ablation = {"per_head_us_per_layer_step": ph_us, "union_us_per_layer_step": ms * 1e3,
                    "union_speedup": ph_us / (ms * 1e3),
                    "kv_tokens_per_head_loading": float(np.sum(own_tok)) / len(layers),
                    "kv_tokens_union": float(np.sum(uni_tok)) / len(layers),
                    "paper": "union up to 1.65x faster than per-head loading (P:695)"}

    # ---- target-fraction sweep (BASELINE.json configs[4], C5): same layers, device-timed
    # like the headline, plus the union fraction the GPU selected
    sweep = []
    if args.sweep and world == 1:
        for p in (0.5, 0.8, 0.9, 0.95, 0.99, 1.0):
            for L in layers:
                L["o_sw"] = torch.empty_like(L["q"])
            gp = model_graph(lambda L: T.decode(L["q"], L["index"], p, out=L["o_sw"]))
            us = 1e3 * tm.timed([gp.replay], max(10, min(args.steps, 50))) / len(layers)
            del gp
            uf = []
            for L in layers:
                if p >= 1.0:
                    uf.append(1.0)
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
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING)"
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    attn_bytes = bm["union_kv"] + bm["q_out"] // 2 + (n_sm + units) * G * 129 * 4   # K/V, q, partials
    att_gbs = attn_bytes / (att_launch_us * 1e-6) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get("attention_kernel_sparse_bytes_per_launch")
    except Exception:
        pass
    import torch.cuda.nccl as tnccl
    line = {
        "metric": METRIC, "value": ms * 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_model_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": _config(args, world),
        # per decode layer-step: score_rank, sample, fit, attention (p < 1); 1 attention at p >= 1
        "gpu_launches": (1 if args.p >= 1 else 4) * LAYERS * args.steps,
        "p50_us": step_p50 * 1e3, "p99_us": step_p99 * 1e3,
        "roofline": {"bound": "hbm", "kernel": "attention_kernel<4,false,true> (S8 sparse split-KV, unit-aligned split + fused S9)",
                     "achieved": att_gbs, "peak": hbm, "unit": "GB/s", "frac": att_gbs / hbm,
                     "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": attn_bytes, "us_per_launch": att_launch_us,
                     "timing": "S8+S9 alone, 8 layers' launches back to back in one graph (no PDL), cold L2 "
                               "per replay, CUDA events; mean per launch (rank 0's units)"},
        "step_roofline": {"bytes_per_step": bm["total"], "achieved_gbs": bm["total"] / (ms * 1e-3) / 1e9,
                          "frac": bm["total"] / (ms * 1e-3) / 1e9 / hbm, "bytes": bm},
        "phases_us": phases,
        "dense": {"us_per_layer_step": dense_ms * 1e3, "gbs_job": dense_bytes / (dense_ms * 1e-3) / 1e9,
                  "frac": dense_bytes / (dense_ms * 1e-3) / 1e9 / hbm / world, "bytes_job": dense_bytes},
        "speedup_vs_dense": dense_ms / ms,
        "isolated_layer_graph": {"us_per_layer_step": iso_us, "dense_us_per_layer_step": dense_iso_ms * 1e3,
                                 "speedup_vs_dense": dense_iso_ms * 1e3 / iso_us,
                                 "what": "each layer-step as its own CUDA graph, L2 flushed before each (includes one graph launch per layer)"},
        "p_sweep": sweep or None,
        "c3": c3,
        "c4": c4,
        "table1": table1,
        "gqa_union_ablation": ablation,
        # ms: the tactic_build_index call bracketed by events (host allocation and launch
        # included); gpu_ms: the library's own events around its kernels (info.build_gpu_ms)
        "build": {"ms": build_ms, "gpu_ms": build_gpu_ms, "units_per_gpu": units, "iters_run": iters_run,
                  "alg_tflop": alg_tflop, "alg_tflops": alg_tflop / (build_gpu_ms * 1e-3),
                  "exec_tflops_split_bf16": 2 * alg_tflop / (build_gpu_ms * 1e-3)},
        "e2e": {"value": e2e_ms * 1e3, "unit": UNIT, "h2d_bytes_per_step": int(layers[0]["q"].numel() * 2),
                "d2h_bytes_per_step": int(layers[0]["q"].numel() * 2),
                "how": "tactic_decode_host per layer-step (pinned q in, decode, out back -- zero-copy: the entry "
                       "kernel reads q from the pinned buffer, the merge writes the output into it; the library "
                       "replays its captured graph), CUDA events around each synchronising call, cold L2; max over "
                       "ranks"},
        "nccl": {"backend": "nccl", "world": world, "version": ".".join(map(str, tnccl.version()))
                 if hasattr(tnccl, "version") else None},
        "clocks": clk.summary(),
        "context": PAPER_CONTEXT,
    }
    if world == 1 and not args.no_cpu_baseline:
        from synth import make_unit
        u = make_unit(n, G, seed=0, b=0, h=0)
        ex = layers[0]["export"]
        line["cpu_baseline"] = cpu_baseline(args, u["K"], u["V"], u["q"], ex["centroids"][0], ex["assign"][0])
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _self_launch(args):
    """`bench.py --gpus N` outside torchrun: re-run under torch.distributed.run, one rank per
    GPU of this node; fails loudly when fewer than N GPUs are visible."""
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}\n")
        sys.exit(2)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines (NVLS, rings) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def same_decode(a, b):
    """Two decodes of the same inputs: equal up to the order of the reference-shift merge's
    fp32 accumulator adds (within two bf16 steps of the larger value: one step can exceed
    2^-7 of the smaller value at a binade boundary)."""
    import torch
    a, b = a.float().cpu(), b.float().cpu()
    ok = bool(torch.all((a - b).abs() <= 2.0 ** -6 * torch.maximum(a.abs(), b.abs()) + 1e-6))
    if not ok:
        d = (a - b).abs()
        i = int(torch.argmax(d))
        print(f"same_decode: max |diff| {float(d.max()):.3e} at {i}: {float(a.flatten()[i]):.6e} vs "
              f"{float(b.flatten()[i]):.6e}", flush=True)
    return ok


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
    ap.add_argument("--c4", type=int, default=1, help="1: add the C4 sequence-sharded step with its collectives")
    ap.add_argument("--ablation", type=int, default=1, help="1: add the GQA union vs per-head loading ablation")
    args = ap.parse_args()
    if args.warmup < 3:
        sys.stderr.write("bench.py: --warmup must be >= 3\n")
        sys.exit(2)
    in_torchrun = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if not in_torchrun and args.gpus > 1:
        _self_launch(args)
        return
    if in_torchrun and world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE\n")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    # one NCCL process group at every world size (world 1 included): barriers, the
    # max-over-ranks reduction of the timings, and the C4 step's collectives
    if in_torchrun:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
