"""Turn one round's gpurun_out/ profiling artefacts into the committed profiles/ summaries.

    python tools/summarize_profiles.py r01

Reads  gpurun_out/bench_<R>.json          (one bench.py JSON line)
       gpurun_out/launches_<R>.csv        (ncu --metrics gpu__time_duration.sum launch list of bench.py)
       gpurun_out/full_<R>.ncu-rep        (ncu --set full of tools/profile_decode.py: one decode + one dense)
       gpurun_out/km_<R>.ncu-rep          (ncu --set full of one tcgen05 k-means assignment launch)
       gpurun_out/km_launches_<R>.csv     (launch list of tools/build_timing.py: 8 C2 layer builds)
Writes profiles/<R>_bench.json, profiles/<R>_launches.txt, profiles/<R>_ncu_full.txt, profiles/<R>_km_build.txt,
       profiles/ncu_traffic.json (dram bytes per launch of the sparse attention kernel, read by bench.py)
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
os.makedirs(PROF, exist_ok=True)

def is_sparse_attention(name):
    """attention_kernel<G, DENSE[, UNIT]> with DENSE = 0 / false (ncu prints either form)."""
    m = re.search(r"attention_kernel<\s*(?:\(int\))?\d+,\s*(?:\(bool\))?(\w+)", name)
    return bool(m) and m.group(1) in ("0", "false")


# ---- bench line
bench_line = None
bp = os.path.join(OUT, f"bench_{R}.json")
if os.path.exists(bp):
    lines = [ln for ln in open(bp).read().splitlines() if ln.startswith("{")]
    if lines:
        bench_line = json.loads(lines[-1])
        json.dump(bench_line, open(os.path.join(PROF, f"{R}_bench.json"), "w"), indent=1)

# ---- launch list: per-kernel count / mean / share of the decode step
lp = os.path.join(OUT, f"launches_{R}.csv")
if os.path.exists(lp):
    rows = list(csv.reader(open(lp)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")) / 1000.0)  # ns -> us
    decode = {k: v for k, v in agg.items()
              if any(s in k for s in ("score_rank", "sample_kernel", "fit_unit")) or is_sparse_attention(k)}
    tot = sum(sum(v) / len(v) for v in decode.values()) or 1.0
    with open(os.path.join(PROF, f"{R}_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list of `python bench.py "
                f"--steps 8 --warmup 3 --no-cpu-baseline --sweep 0 --c3 0 --table1 0 --ablation 0 --c4 0` ({R}).\n# Per-launch times are cold-cache and "
                f"serialised (no PDL overlap): compare shares, not absolutes.\n")
        f.write(f"{'launches':>8} {'mean us':>9} {'share of decode':>16}  kernel\n")
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            m = sum(v) / len(v)
            share = f"{m / tot * 100:15.1f}%" if k in decode else " " * 16
            f.write(f"{len(v):8d} {m:9.2f} {share}  {k[:110]}\n")
        f.write(f"\n# decode kernels (one step): {tot:.2f} us summed serialised\n")

# ---- ncu --set full: key metrics per kernel
fp = os.path.join(OUT, f"full_{R}.ncu-rep")
if os.path.exists(fp):
    raw = subprocess.run(["ncu", "-i", fp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
            ("dram__bytes_write.sum", "dram write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
            ("launch__grid_size", "grid"), ("launch__block_size", "block"),
            ("launch__registers_per_thread", "regs"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %")]
    idx = {m: h.index(m) for m, _ in want if m in h}
    traffic = {}
    with open(os.path.join(PROF, f"{R}_ncu_full.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none of tools/profile_decode.py (C2: 128K tokens, 8 KV heads, "
                f"G=4, C=1024, p=0.9): one decode (score_rank, sample, fit, sparse attention) + one dense decode "
                f"({R}).\n")
        for r in rr[2:]:
            name = r[h.index("Kernel Name")]
            f.write(f"\n{name[:120]}\n")
            for m, lab in want:
                if m in idx:
                    f.write(f"  {lab:16s} {r[idx[m]]:>14s} {units[idx[m]]}\n")
            if "attention_kernel" in name and "dram__bytes_read.sum" in idx:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(r[idx["dram__bytes_read.sum"]]) * scale.get(units[idx["dram__bytes_read.sum"]], 1)
                wr = float(r[idx["dram__bytes_write.sum"]]) * scale.get(units[idx["dram__bytes_write.sum"]], 1)
                key = "sparse" if is_sparse_attention(name) else "dense"
                traffic[f"attention_kernel_{key}_bytes_per_launch"] = rd + wr
        # stall breakdown per kernel from the source page
        f.write("\n# warp-stall reasons (share of samples) per kernel\n")
        src = subprocess.run(["ncu", "-i", fp, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        blocks, cur = [], None
        for ln in src.splitlines():
            if ln.startswith('"Kernel Name"'):
                cur = [ln]
                blocks.append(cur)
            elif cur is not None:
                cur.append(ln)
        seen = set()
        for b in blocks:
            if b[0] in seen:
                continue
            seen.add(b[0])
            rows = list(csv.reader(b[1:]))
            if not rows:
                continue
            hh = rows[0]
            cols = [i for i, x in enumerate(hh) if x.startswith("stall_") and "Not Issued" not in x]
            agg = collections.Counter()
            for row in rows[1:]:
                for i in cols:
                    try:
                        agg[hh[i][6:]] += float(row[i] or 0)
                    except (ValueError, IndexError):
                        pass
            t = sum(agg.values()) or 1
            f.write(f"{b[0].split(',', 1)[1][:90]}: " + " ".join(f"{k}={v / t * 100:.0f}%"
                                                               for k, v in agg.most_common(6)) + "\n")
    if traffic:
        traffic["source"] = f"profiles/{R}_ncu_full.txt (dram__bytes_read.sum + dram__bytes_write.sum)"
        json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
# ---- index build: tcgen05 assignment capture + the build's launch list
kp, klp = os.path.join(OUT, f"km_{R}.ncu-rep"), os.path.join(OUT, f"km_launches_{R}.csv")
if os.path.exists(kp) or os.path.exists(klp):
    with open(os.path.join(PROF, f"{R}_km_build.txt"), "w") as f:
        f.write(f"# C2 index build (8 units x 131072 keys, C = 1024, 10 Lloyd iterations) ({R}).\n")
        if os.path.exists(klp):
            rows = list(csv.reader(open(klp)))
            hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
            h = rows[hi]
            ki, vi = h.index("Kernel Name"), h.index("Metric Value")
            agg = collections.defaultdict(list)
            for r in rows[hi + 1:]:
                if len(r) > vi:
                    agg[r[ki]].append(float(r[vi].replace(",", "")) / 1000.0)
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
                    "`python tools/build_timing.py --layers 8` (cold, serialised; the first build is a warm-up "
                    "of 8192 keys):\n")
            f.write(f"{'launches':>8} {'mean us':>9}  kernel\n")
            for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
                f.write(f"{len(v):8d} {sum(v) / len(v):9.2f}  {k[:100]}\n")
        if os.path.exists(kp):
            raw = subprocess.run(["ncu", "-i", kp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rr = list(csv.reader(io.StringIO(raw)))
            h, units = rr[0], rr[1]
            f.write("\n# ncu --set full --clock-control none of one km_assign_tc_kernel launch "
                    "(tools/profile_build.py, 4th assignment):\n")
            for m in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                      "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
                      "l1tex__m_xbar2l1tex_read_bytes.sum.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                      "dram__bytes_read.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread"):
                if m in h:
                    f.write(f"  {m:70s} {rr[2][h.index(m)]:>12s} {units[h.index(m)]}\n")
# ---- C3 launch list (tools/profile_c3.py: 3 decodes + 1 dense decode, batch 64 x 32K)
cp = os.path.join(OUT, f"c3_launches_{R}.csv")
if os.path.exists(cp):
    rows = list(csv.reader(open(cp)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")) / 1000.0)
    with open(os.path.join(PROF, f"{R}_c3_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
                f"`python tools/profile_c3.py` ({R}): C3 = batch 64 x 8 KV heads x 32K tokens (512 units), "
                f"C = 256, p = 0.9; 3 sparse decodes + 1 dense decode, cold L2 (ncu flushes).\n")
        f.write(f"{'launches':>8} {'mean us':>9}  kernel\n")
        for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
            f.write(f"{len(v):8d} {sum(v) / len(v):9.2f}  {k[:110]}\n")
print(open(os.path.join(PROF, f"{R}_launches.txt")).read() if os.path.exists(lp) else "no launch list")
