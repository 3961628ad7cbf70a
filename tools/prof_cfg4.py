"""Stage times of the fKK-EC transform on a cfg4-geometry row block (M = 1600, k = 100: 13 image blocks, the
one-CTA Gram path) -- python tools/prof_cfg4.py [rows] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS["cfg4"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True)
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
acc = {}
for r in range(reps + 1):
    plan.transform(I, R, out)
    if r:
        for k, v in plan.stage_times().items():
            acc[k] = acc.get(k, 0.0) + v / reps
torch.cuda.synchronize()
print(f"cfg4 geometry, {rows} rows: stages {acc}")
