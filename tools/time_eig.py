"""Time the fKK-EC stages on cfg3 (one plan, a few steps) -- quick A/B of kernel changes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
I, R, _ = generate_rows(cfg, 0, cfg.n_pixels)
Id, Rd = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, cfg.n_pixels, timing=True)
out = torch.empty((cfg.n_pixels, cfg.n_freq), dtype=torch.complex64, device="cuda")
acc = {}
for it in range(4):
    plan.transform(Id, Rd, out)
    if it >= 1:
        for k, v in plan.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v / 3
print(json.dumps({k: round(v, 3) for k, v in acc.items()}), "total", round(sum(acc.values()), 3))
