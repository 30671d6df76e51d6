"""In-kernel %globaltimer stamps of the decode kernels on the C2 workload (TACTIC_TLOG=1).

    python tools/phase_timing.py [--no-flush]
Debug aid only: prints the kernel timeline, the score_rank / fit phases and CTA 0 of the
attention kernel (setup, tiles issued / consumed, merges), relative times in us.
"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between calls")
ap.add_argument("--c3", action="store_true", help="C3 workload (batch 64, 32K, C = 256) instead of C2")
args = ap.parse_args()
os.environ["TACTIC_TLOG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402
from synth import make_layer  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

if args.c3:
    import bench  # noqa: E402
    G, n, C = 4, 32768, 256
    L = bench.make_layers([9000], torch.device("cuda", 0), [(b, h) for b in range(64) for h in range(8)], n=n)[0]
    Kd, Vd, qd = L["K"], L["V"], L["q"]
    idx = T.build_index(Kd, Vd, C, 10, group_size=G, seed=9000)
else:
    G, n, C = 4, 131072, 1024
    K, V, q = make_layer(1, 8, G, n, seed=0)
    to = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
    Kd, Vd, qd = to(K), to(V), to(q)
    idx = T.build_index(Kd, Vd, C, 10, group_size=G)
R = 0  # multi-kernel selection (the only path)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty_like(qd)
T.decode(qd, idx, 0.9, out=out)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()  # replayed like bench.py (no host launch gaps)
with torch.cuda.graph(graph):
    T.decode(qd, idx, 0.9, out=out)
for it in range(4):
    if not args.no_flush:
        flush.fill_(1)
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    full = idx.debug_timing().astype(np.int64).reshape(-1)
    acc_now = full[2100:2700].copy()  # per-CTA accumulators: report this call's increment
    if it > 0:
        full[2100:2700] -= acc_prev
    acc_prev = acc_now
    if it < 2:
        continue
    print(f"--- iteration {it}")
    tl = full[1536:1536 + 20].reshape(5, 4)
    if (tl[:, 0] > 0).any():
        z = tl[:, 0][tl[:, 0] > 0].min()
        print("  timeline (us from first start: first-CTA start / past wait / last CTA end):")
        for k, nm in enumerate(["score", "score+rank", "sample", "fit", "attention"]):
            if tl[k, 0] > 0:
                print(f"    {nm:9s} {(tl[k, 0] - z) / 1e3:7.2f} {(tl[k, 1] - z) / 1e3:7.2f} {(tl[k, 2] - z) / 1e3:7.2f}")
        se = full[3000:3512].reshape(-1, 2)
        live = se[:, 0] > 0
        if live.any():
            st, en = (se[live, 0] - z) / 1e3, (se[live, 1] - z) / 1e3
            print(f"  score_rank CTAs: start min {st.min():.2f} max {st.max():.2f}; end min {en.min():.2f} "
                  f"median {np.median(en):.2f} max {en.max():.2f}; dur min {(en - st).min():.2f} median "
                  f"{np.median(en - st):.2f} max {(en - st).max():.2f}")
            ids = np.nonzero(live)[0]
            order = np.argsort(-en)[:6]
            rkd = (full[4096:4096 + len(live)][live].astype(np.int64) - z) / 1e3
            print("   slowest (cta, start, ranked, end): " + ", ".join(f"({ids[i]}, {st[i]:.2f}, {rkd[i]:.2f}, {en[i]:.2f})" for i in order))
            print(f"   ranked: min {rkd.min():.2f} median {np.median(rkd):.2f} max {rkd.max():.2f}; rowmap phase (end - ranked): "
                  f"median {np.median(en - rkd):.2f} max {(en - rkd).max():.2f}")
        sp = full[4608:4608 + 4 * 880].reshape(-1, 4).astype(np.int64)
        lv = sp[:, 3] > 0
        if lv.any():
            sp = (sp[lv] - z) / 1e3
            print(f"  sample CTAs ({int(lv.sum())}): start min {sp[:,0].min():.2f} max {sp[:,0].max():.2f}; past wait min "
                  f"{sp[:,1].min():.2f} max {sp[:,1].max():.2f}; rows in (after wait) median {np.median(sp[:,2]-sp[:,1]):.2f} "
                  f"max {(sp[:,2]-sp[:,1]).max():.2f}; end min {sp[:,3].min():.2f} median {np.median(sp[:,3]):.2f} max {sp[:,3].max():.2f}")
            late = np.argsort(-sp[:, 3])[:5]
            print("   latest (start, wait, rows, end):", [tuple(np.round(sp[i], 2).tolist()) for i in late])
        rk = full[1600:1607]
        if rk[0] > 0:
            names = ["centroids in", "scored", "sorted", "pushed", "runs in", "ranked", "rowmap"]
            print("  rank CTA(0,0) phases (us after its wait): " +
                  "  ".join(f"{nm} {(rk[i] - tl[1, 1]) / 1e3:.2f}" for i, nm in enumerate(names)))
    if R == 0 and full[256] > 0 and full[256 + 6] == 0:
        fs = full[256:256 + 6]
        z = tl[:, 0][tl[:, 0] > 0].min()
        names = ["head0 last chunk", "staged", "fitted", "marked", "unit0 compact start", "unit0 compact end"]
        print("  sample_fit (us from first start): " + "  ".join(f"{nm} {(fs[i] - z) / 1e3:6.2f}" for i, nm in enumerate(names)
                                                              if fs[i] > 0))
        ds = full[270:274]
        if ds[0] > 0:
            print("  fit unit 0 descriptors (us from first start): " + "  ".join(
                f"{nm} {(x - z) / 1e3:.2f}" for nm, x in zip(["arrived", "all arrived", "totals", "written"], ds)))
        hw = full[2720:2720 + 64].reshape(8, 8)
        for g in range(8):
            if hw[g, 0] > 0:
                print(f"   fit head {g} (us after staged): " + "  ".join(
                    f"{nm} {(hw[g, i] - full[256 + 2]) / 1e3:.2f}" for i, nm in
                    [(0, "sums"), (1, "W"), (3, "J"), (4, "marked")] if hw[g, i] > 0) +
                    f"  path {'exact-head' if hw[g, 7] == 1 else 'tail' if hw[g, 7] == 2 else '-'}")
        hs = full[1700:1705]
        if hs[0] > 0:
            print("  fit warp 0 (us after summaries staged): " + "  ".join(
                f"{nm} {(hs[i] - fs[2]) / 1e3:.2f}" for i, nm in enumerate(["sums", "W", "-", "J", "marked"]) if hs[i] > 0))
        cf = full[1720:1725]
        print("  fit CTA u0 clock64 cycles: staged->marked %d  marked->lists %d" % (cf[3] - cf[2], cf[4] - cf[3]))
        cr = full[1730:1734]
        if cr[0] > 0:
            print("  fit mask lists, cycles per repetition:", np.diff(cr).tolist())
        cc = full[1740:1745].astype(np.int64)
        if cc[0] > 0:
            print("  fit compaction (clock64 cycles, thread 0 of unit 0): loc+scan %d  w_sum sync %d  base+lists %d  padding %d"
                  % (cc[1] - cc[0], cc[2] - cc[1], cc[3] - cc[2], cc[4] - cc[3]))
        cs = full[264:268]
        print("  compaction (us from first start): " + "  ".join(f"{nm} {(cs[i] - z) / 1e3:6.2f}" for i, nm in
              enumerate(["pass1", "scan", "pass2", "fill"]) if cs[i] > 0))
        t0 = z
    elif R == 0:
        fs = full[256:256 + 7]
        t0 = fs[0]
        names = ["start", "pdl_wait", "staged", "heads fitted", "compacted", "last-unit start", "last-unit end"]
        print("  fit CTA u0: " + "  ".join(f"{nm} {(fs[i] - t0) / 1e3:6.2f}" for i, nm in enumerate(names)
                                             if fs[i] > 0))
        hs = full[1700:1705]
        if hs[0] > 0:
            names = ["sums", "W", "k*", "J", "marked"]
            print("  fit warp 0 (us after staged): " + "  ".join(f"{nm} {(hs[i] - fs[2]) / 1e3:.2f}"
                                                               for i, nm in enumerate(names) if hs[i] > 0))
            ck = full[1709:1715]
            print("  fit warp 0 (cycles after staged): " + "  ".join(f"{nm} {ck[i + 1] - ck[0]}" for i, nm in enumerate(names) if hs[i] > 0))
    at = full[192:192 + 35]
    if at[0] > 0:
        b0 = at[0]
        iss = [(x - b0) / 1e3 for x in at[2:18] if x > 0]
        con = [(x - b0) / 1e3 for x in at[18:34] if x > 0]
        print(f"  attention CTA0: starts {(b0 - t0) / 1e3:.2f} us after selection start; ends +{(at[34] - b0) / 1e3:.2f}")
        print("   tiles issued at", np.round(iss, 2).tolist())
        pz = full[192 + 40:192 + 49]
        print("   producer setup (us after wait): " + "  ".join(f"{nm} {(x - b0) / 1e3:.2f}" for nm, x in
              zip(["split", "lists loaded", "synced", "search start", "window in", "all lists in", "split rep0", "split rep1", "split rep2"], pz) if x > 0))
        print("   tiles consumed at", np.round(con, 2).tolist())
        ce = full[512:512 + 296].reshape(-1, 2)
        ce = ce[(ce[:, 0] > 0) & (ce[:, 1] > 0)]
        if len(ce):
            st, en = (ce[:, 0] - b0) / 1e3, (ce[:, 1] - b0) / 1e3
            print(f"   all CTAs: start min {st.min():.2f} max {st.max():.2f}; end min {en.min():.2f} "
                  f"median {np.median(en):.2f} max {en.max():.2f}; slowest CTA {int(np.argmax(en))}")
            nt_ = full[816:816 + 148]
            order = np.argsort(-en)[:8]
            print("   slowest CTAs (cta, end us, tiles):", [(int(c), round(float(en[c]), 2), int(nt_[c])) for c in order])
            print("   tiles per CTA: min %d median %d max %d" % (nt_.min(), np.median(nt_), nt_.max()))
            pe = full[2100:2248] / 1e3
            nm_ = full[2300:2448]
            npc_ = full[2500:2648]
            print("   piece-end us per CTA: min %.2f median %.2f max %.2f; merges per CTA: min %d median %d max %d; "
                  "pieces per CTA: median %d" % (pe.min(), np.median(pe), pe.max(), nm_.min(), np.median(nm_), nm_.max(),
                                                 np.median(npc_)))
            print("   slowest CTAs (cta, end, piece-end us, merges, pieces):",
                  [(int(c), round(float(en[c]), 1), round(float(pe[c]), 2), int(nm_[c]), int(npc_[c])) for c in order])
            fast = np.argsort(en)[:5]
            print("   fastest CTAs (cta, end, piece-end us, merges, pieces, tiles):",
                  [(int(c), round(float(en[c]), 1), round(float(pe[c]), 2), int(nm_[c]), int(npc_[c]), int(nt_[c])) for c in fast])
            meta = full[3600:3748]
            rel = full[3800:3948]
            if (rel > 0).any():
                uu = (meta & 0xFFFF).astype(int)
                jj = ((meta >> 16) & 0xFFFF).astype(int)
                print("   per unit: CTAs, slowest piece arrival (non-merger), merger poll done, merger end (us):")
                for uni in sorted(set(uu.tolist())):
                    cs = [c for c in range(148) if uu[c] == uni and rel[c] > 0]
                    nm = [c for c in cs if jj[c] != 0]
                    mc = [c for c in cs if jj[c] == 0]
                    sl = max(((rel[c] - b0) / 1e3 for c in nm), default=float('nan'))
                    md = ((rel[mc[0]] - b0) / 1e3) if mc else float('nan')
                    me = (en[mc[0]]) if mc else float('nan')
                    tk = full[5200:5348]
                    tks = [int(tk[c]) for c in nm] or [0]
                    print(f"     unit {uni}: {len(cs)} CTAs, tokens per CTA {min(tks)}-{max(tks)} (merger {int(tk[mc[0]]) if mc else -1}), "
                          f"slowest arrival {sl:.2f}, merger poll {md:.2f}, merger end {me:.2f}")
            nr = full[5400:5548].astype(np.int64)
            tk = full[5200:5348].astype(np.int64)
            if (rel > 0).any() and nr.sum() > 0:
                arr = (rel.astype(np.int64) - b0) / 1e3
                ok = (rel > 0) & (tk > 0)
                c = np.corrcoef(np.vstack([arr[ok], nr[ok], tk[ok]]))
                print(f"   per CTA: runs min {nr[ok].min()} median {int(np.median(nr[ok]))} max {nr[ok].max()}; "
                      f"corr(arrival, runs) {c[0,1]:.2f}, corr(arrival, tokens) {c[0,2]:.2f}")
                slow = np.argsort(-np.where(ok, arr, -1))[:6]
                print("   slowest arrivals (cta, arrival, tokens, runs):", [(int(i), round(float(arr[i]), 2), int(tk[i]), int(nr[i])) for i in slow])
                fastc = np.argsort(np.where(ok, arr, 1e9))[:6]
                print("   fastest arrivals (cta, arrival, tokens, runs):", [(int(i), round(float(arr[i]), 2), int(tk[i]), int(nr[i])) for i in fastc])
            mg = full[964:964 + 16].reshape(8, 2)
            print("   merges (start, end) us:", [(round((s - b0) / 1e3, 2), round((e - b0) / 1e3, 2)) for s, e in mg if s > 0])
            cp = full[980:988]
            npc = full[990:998]
            print("   merge staged at / pieces:", [(round((c - b0) / 1e3, 2), int(k)) for c, k in zip(cp, npc) if c > 0])
