"""Shared helpers for the GPU parity tests (inputs from synth/, expectations from oracle/)."""
import numpy as np
import torch

from oracle import tactic_oracle as O

TOL_MAX_ABS = 2e-2      # BASELINE.json north_star: decode output, bf16 KV
TOL_REL_L2 = 5e-3
TOL_THRESHOLD = 1e-5    # index-set mismatch allowed only within 1e-5 of the threshold


def dev_bf16(a: np.ndarray) -> torch.Tensor:
    """float32 array holding bf16-representable values -> CUDA bf16 tensor (exact)."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda").to(torch.bfloat16)


def rel_l2(x: np.ndarray, y: np.ndarray) -> float:
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30))


def assert_output_close(got: np.ndarray, ref: np.ndarray, what: str = ""):
    ma = float(np.max(np.abs(got - ref)))
    rl = rel_l2(got, ref)
    assert ma <= TOL_MAX_ABS and rl <= TOL_REL_L2, f"{what}: max-abs {ma:.3e} rel-L2 {rl:.3e}"
    return ma, rl


def assert_same_decode(a: torch.Tensor, b: torch.Tensor, what: str = ""):
    """Two decodes of the same inputs in the default merge: the reference-shift merge adds
    the pieces' shares with fp32 atomics, so outputs may differ by fp32 summation order --
    within two bf16 steps of the larger value (one step can exceed 2^-7 of the smaller one
    at a binade boundary; OPT_DETERMINISTIC: bit-identical)."""
    x, y = a.float().cpu(), b.float().cpu()
    bad = (x - y).abs() > 2.0 ** -6 * torch.maximum(x.abs(), y.abs()) + 1e-6
    assert not bool(bad.any()), f"{what}: {int(bad.sum())} elements differ by more than two bf16 steps"


def oracle_layer_clustering(K, V, C, iters, seed):
    """Per-unit oracle k-means over a [B][H][n][d] layer; returns centroids, assign, indices."""
    B, H, n, d = K.shape
    cents, asg, idxs = [], [], []
    for b in range(B):
        for h in range(H):
            u = b * H + h
            idx, km = O.build_index(K[b, h], V[b, h], C, iters, seed=seed, unit=u)
            cents.append(km["centroids"].astype(np.float32))
            asg.append(km["assign"].astype(np.int32))
            idxs.append(idx)
    return np.stack(cents), np.stack(asg), idxs


def j_mismatch_allowed(head: dict, Jg: int, p: float) -> bool:
    """A J difference is allowed only if every cluster end between the two J lies within
    TOL_THRESHOLD of the threshold (oracle's estimated cumulative mass)."""
    Jo = head["J"]
    if Jg == Jo:
        return True
    lo, hi = min(Jg, Jo), max(Jg, Jo)
    ce = head["cum_end"] / head["W"]
    return all(abs(ce[r - 1] - p) < TOL_THRESHOLD for r in range(lo, hi))
