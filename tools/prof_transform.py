"""One fKK-EC transform of a cfg3 row block (default: the full image) for ncu captures.
   python tools/prof_transform.py [rows] [reps] [svd]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS["cfg3"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_pixels
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
svd = sys.argv[3] if len(sys.argv) > 3 else "gram"
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True, svd=svd)
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
for _ in range(reps):
    plan.transform(I, R, out)
torch.cuda.synchronize()
print(f"transform {rows} rows ({svd}): stages {plan.stage_times()}")
