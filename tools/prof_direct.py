"""Run the direct path (kk_direct_batch) on a cfg3 row block for ncu / timing: a plan without stage
events, then one with them (the per-stage split).
   python tools/prof_direct.py [rows] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS["cfg3"]
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
for timing in (False, True):
    plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=timing)
    plan.als_solves()
    plan.direct(I, R, out)
    torch.cuda.synchronize()
    solves = plan.als_solves() / rows
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.direct(I, R, out)
    e1.record()
    torch.cuda.synchronize()
    extra = f"; stages {plan.stage_times()}" if timing else ""
    print(f"direct {rows} rows ({'stage events' if timing else 'no stage events'}): "
          f"{e0.elapsed_time(e1) / reps:.3f} ms/pass; ALS solves/spectrum {solves:.3f}{extra}")
    del plan
