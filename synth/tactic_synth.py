"""tactic-synth-v1: seeded synthetic Q/K/V shaped like Llama-3-8B attention heads.

This module is INPUT GENERATION ONLY.  It holds none of Tactic's arithmetic
(no clustering, scoring, fitting, selection or attention); both the CPU oracle
(`oracle/`) and the CUDA path consume the tensors it returns, so neither side
can leak into the other through it.

Recipe (restated in DESIGN.md "Input recipe"):

* Latent structure: L = max(1, n // 128) latent centres mu_l ~ N(0, I_d);
  token -> latent assignment in geometric runs (mean length 16) of uniformly
  random latent ids -- positional discontinuity as in the paper's t-SNE of keys
  (§3.6 Fig. 6).
* Keys: k_i = mu_{z_i} + 0.5 eps_i + 2 sqrt(d) m_hat (m_hat a unit "common key
  offset" direction).  Sink tokens (positions 0-3 plus n//256 - 4 random
  "delimiter" positions) have k = sqrt(d) u_hat + 0.05 eps with u_hat ⟂ m_hat
  and no offset, i.e. a distinct key group (SURVEY §8(c) reading 21).
* Queries (G per KV head): A = 4 hot latents per head, each shared group-wide
  with probability 0.9, else head-specific.  q_g is the least-norm vector
  meeting the expected-logit targets (q.k/sqrt(d)): hot latent of rank r gets
  8 - ln(r) + 0.5 N(0,1); sinks 7.5; the common offset contributes -1.  An
  isotropic component orthogonal to those constraints adds logit std 0.35.
  This yields heavy-tailed scores with an attention sink (PAPER.md P:189,
  P:313-327, Fig. 7).
* Values: random unit directions x (1 + 0.05 N(0,1)) -- near-constant norm as
  in the paper's Fig. 2.
* Precision: every tensor is rounded to bfloat16 (round-to-nearest-even) and
  returned as float32 arrays holding exactly bf16-representable values, plus
  helpers that return the raw uint16 bf16 bit patterns.

Everything is a pure function of (seed, b, h, n, d, G).
"""
from __future__ import annotations

import numpy as np

D_HEAD = 128
RECIPE = "tactic-synth-v1"


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of float32 values that are already bf16-representable."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def _unit_rng(seed: int, b: int, h: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(b), int(h), 0x7AC71C]))


def _geometric_runs(rng: np.random.Generator, n: int, L: int, mean_run: float = 16.0) -> np.ndarray:
    z = np.empty(n, dtype=np.int64)
    pos = 0
    # draw runs in batches for speed
    while pos < n:
        lens = rng.geometric(1.0 / mean_run, size=max(64, (n - pos) // int(mean_run) + 64))
        ids = rng.integers(0, L, size=lens.shape[0])
        for ln, lid in zip(lens, ids):
            if pos >= n:
                break
            e = min(n, pos + int(ln))
            z[pos:e] = lid
            pos = e
    return z


def make_unit(n: int, G: int = 4, seed: int = 0, b: int = 0, h: int = 0, d: int = D_HEAD,
              n_hot: int = 4, share_prob: float = 0.9):
    """One (sequence b, KV head h) unit.  Returns dict of float32 arrays (bf16 values):
    K [n][d], V [n][d], q [G][d], plus metadata (sink positions, latent ids)."""
    if n < 1 or G < 1 or d < 2:
        raise ValueError("n, G must be >= 1 and d >= 2")
    rng = _unit_rng(seed, b, h)
    sd = np.sqrt(d)
    L = max(1, n // 128)
    mu = rng.standard_normal((L, d))
    # orthonormal offset / sink directions
    m_hat = rng.standard_normal(d)
    m_hat /= np.linalg.norm(m_hat)
    u_hat = rng.standard_normal(d)
    u_hat -= (u_hat @ m_hat) * m_hat
    u_hat /= np.linalg.norm(u_hat)

    z = _geometric_runs(rng, n, L)
    eps = rng.standard_normal((n, d), dtype=np.float32)
    K = mu[z].astype(np.float32) + np.float32(0.5) * eps + np.float32(2.0 * sd) * m_hat.astype(np.float32)

    n_sink = max(min(4, n), n // 256)
    sinks = list(range(min(4, n)))
    if n_sink > len(sinks):
        extra = rng.choice(np.arange(4, n), size=n_sink - len(sinks), replace=False)
        sinks += sorted(int(x) for x in extra)
    sinks = np.array(sinks, dtype=np.int64)
    K[sinks] = (sd * u_hat).astype(np.float32) + np.float32(0.05) * rng.standard_normal((len(sinks), d), dtype=np.float32)

    # values: random unit directions with near-constant norm
    V = rng.standard_normal((n, d), dtype=np.float32)
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    V *= (1.0 + 0.05 * rng.standard_normal((n, 1))).astype(np.float32)

    # queries
    shared = rng.choice(L, size=min(n_hot, L), replace=False)
    q = np.zeros((G, d))
    for g in range(G):
        hot = []
        for a in range(len(shared)):
            if rng.random() < share_prob:
                hot.append(int(shared[a]))
            else:
                hot.append(int(rng.integers(0, L)))
        hot = list(dict.fromkeys(hot))  # distinct, keep order
        rows, tgt = [], []
        for r, l in enumerate(hot, start=1):
            rows.append((mu[l] + 2.0 * sd * m_hat) / sd)
            tgt.append(8.0 - np.log(r) + 0.5 * rng.standard_normal())
        rows.append(u_hat)            # sink: q.(sqrt(d) u)/sqrt(d)
        tgt.append(7.5)
        rows.append(2.0 * m_hat)      # common offset: q.(2 sqrt(d) m)/sqrt(d)
        tgt.append(-1.0)
        M = np.array(rows)
        t = np.array(tgt)
        qg = M.T @ np.linalg.solve(M @ M.T, t)
        # isotropic component orthogonal to the constraint rows, logit std 0.35
        Qm, _ = np.linalg.qr(M.T)
        r = rng.standard_normal(d)
        r -= Qm @ (Qm.T @ r)
        r /= max(np.linalg.norm(r), 1e-12)
        sigma = np.sqrt(1.25)  # per-dim std of background keys around their centre
        qg += r * (0.35 * sd / sigma)
        q[g] = qg
    return {
        "K": bf16_round(K), "V": bf16_round(V), "q": bf16_round(q.astype(np.float32)),
        "sinks": sinks, "latent": z, "n": n, "G": G, "d": d,
    }


def make_layer(B: int, Hkv: int, G: int, n: int, seed: int = 0, d: int = D_HEAD):
    """A Llama-shaped layer: K,V [B][Hkv][n][d], q [B][Hkv*G][d] (float32 arrays of bf16 values).
    Query head j of sequence b belongs to KV head j // G (GQA)."""
    K = np.empty((B, Hkv, n, d), dtype=np.float32)
    V = np.empty((B, Hkv, n, d), dtype=np.float32)
    q = np.empty((B, Hkv * G, d), dtype=np.float32)
    for b in range(B):
        for h in range(Hkv):
            u = make_unit(n, G, seed, b, h, d)
            K[b, h] = u["K"]
            V[b, h] = u["V"]
            q[b, h * G:(h + 1) * G] = u["q"]
    return K, V, q


def uniform_unit(n: int, G: int, seed: int, d: int = D_HEAD, scale: float = 1.0):
    """Plain i.i.d. Gaussian unit (edge-case tests: flat attention, weak clustering)."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 0x0F1A7]))
    K = bf16_round((scale * rng.standard_normal((n, d))).astype(np.float32))
    V = bf16_round(rng.standard_normal((n, d)).astype(np.float32))
    q = bf16_round((scale * rng.standard_normal((G, d))).astype(np.float32))
    return {"K": K, "V": V, "q": q, "n": n, "G": G, "d": d}


# Named workloads (BASELINE.json configs).  Only shapes live here.
CONFIGS = {
    "C1": dict(B=1, Hkv=1, G=4, n=4096, C=64, p=0.9),
    "C2": dict(B=1, Hkv=8, G=4, n=131072, C=1024, p=0.9),
    "C3": dict(B=64, Hkv=8, G=4, n=32768, C=256, p=0.9),
    "C4": dict(B=1, Hkv=8, G=4, n=1048576, C=1024, p=0.9, shards=8),
}
