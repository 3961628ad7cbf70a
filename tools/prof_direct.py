"""Run the direct path (kk_direct_batch) once on a cfg3 row block for ncu / timing.
   python tools/prof_direct.py [rows] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_07132_b200 import fkk
from synth import CONFIGS, generate_rows
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS["cfg3"]
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True)
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
plan.als_solves()
plan.direct(I, R, out)
torch.cuda.synchronize()
print(f"ALS solves per spectrum: {plan.als_solves() / rows:.3f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    plan.direct(I, R, out)
e1.record(); torch.cuda.synchronize()
print(f"direct {rows} rows: {e0.elapsed_time(e1)/reps:.3f} ms/pass; stages {plan.stage_times()}")
