"""Streaming bandwidth of the dense flash-decode kernel vs CTA count (C2 cache, 537 MB):
how much HBM bandwidth a subset of the SMs can pull (sizing the one-launch decode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_12216_b200 import build as B  # noqa: E402

B.build()
from paper_2502_12216_b200 import tactic as T  # noqa: E402

n, H, G = 131072, 8, 4
K = torch.randn(1, H, n, 128, device="cuda").to(torch.bfloat16)
V = torch.randn(1, H, n, 128, device="cuda").to(torch.bfloat16)
q = torch.randn(1, H * G, 128, device="cuda").to(torch.bfloat16)
for ctas in [8, 16, 32, 64, 96, 128, 148, 296]:
    out = T.dense_decode(q, K, V, num_ctas=ctas)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        T.dense_decode(q, K, V, out=out, num_ctas=ctas)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    gbs = 2 * K.numel() * 2 / us / 1e3
    print(f"ctas {ctas:4d}: {us:8.1f} us  {gbs:7.0f} GB/s  {gbs / ctas:6.1f} GB/s per CTA", flush=True)
