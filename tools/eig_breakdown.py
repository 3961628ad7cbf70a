"""Per-kernel device times of the GPU eigensolver (fkk_debug_eig_topk) via the CUPTI activity
records of torch.profiler -- quick A/B of eig kernel changes (not a bench number)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rng = np.random.default_rng(0)
lam = np.concatenate([np.geomspace(1e4, 1.0, 16), np.linspace(0.9, 0.5, M - 16)])
Q, _ = np.linalg.qr(rng.standard_normal((M, M)))
G = torch.from_numpy((Q * lam) @ Q.T).cuda()
G = 0.5 * (G + G.T).contiguous()
for _ in range(2):
    fkk.fkk_debug_eig_topk(G, k)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        fkk.fkk_debug_eig_topk(G, k)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        n = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        tot[n] = tot.get(n, 0.0) + e.device_time_total / 3 / 1e3
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.3f} ms  {n}")
print(f"{sum(tot.values()):9.3f} ms  total (M={M}, k={k})")
