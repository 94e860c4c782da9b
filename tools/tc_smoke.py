"""Quick correctness probe of the tcgen05 attention kernel vs the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_16481_b200 as F  # noqa: E402
from oracle import restated as O  # noqa: E402

r = np.random.default_rng(0)
for d, H, m in ((64, 4, 100), (32, 2, 16), (64, 4, 300), (96, 4, 777), (128, 1, 200), (512, 4, 1000),
                (48, 2, 129), (256, 2, 64)):
    Q, K, V = (r.normal(size=(m + 20, d)) for _ in range(3))
    rg = [(5, 5 + m // 2), (10 + m // 2, 10 + m)]
    out = F.tiled_attention(Q, K, V, F.AttentionParams(d, H), ranges=rg)
    torch.cuda.synchronize()
    ref = O.attention_ranges(Q, K, V, H, rg)
    rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    print(f"d={d} H={H} m={m} rel={rel:.3e}", flush=True)
