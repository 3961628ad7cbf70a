"""Stage timing of the cfg3 transform (the eig stage and the rest): mean stage split over `reps` transforms after a warm-up
(plan stage events).  python tools/time_eig.py [rows] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS["cfg3"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_pixels
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True)
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
plan.transform(I, R, out)
torch.cuda.synchronize()
acc = {}
for _ in range(reps):
    plan.transform(I, R, out)
    torch.cuda.synchronize()
    for k, v in plan.stage_times().items():
        acc[k] = acc.get(k, 0.0) + v / reps
print("stages " + ", ".join(f"{k} {v:.3f}" for k, v in acc.items())
      + f"; total {sum(acc.values()):.3f} ms")
