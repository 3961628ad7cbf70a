"""Per-kernel device times (CUPTI via torch.profiler) of one fKK-EC transform, one direct-KK pass or
one ML apply on a workload's first N rows -- quick A/B of kernel changes (not a bench number)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--what", default="direct", choices=["direct", "transform"])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.workload]
n = a.rows or cfg.n_pixels
I, R, _ = generate_rows(cfg, 0, n)
Id, Rd = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, n)
out = torch.empty((n, cfg.n_freq), dtype=torch.complex64, device="cuda")
run = (lambda: plan.direct(Id, Rd, out)) if a.what == "direct" else (lambda: plan.transform(Id, Rd, out))
run()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        run()
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        nm = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        tot[nm] = tot.get(nm, 0.0) + e.device_time_total / a.reps / 1e3
for nm, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{v:9.3f} ms  {nm}")
print(f"{sum(tot.values()):9.3f} ms  total ({a.what}, {a.workload}, {n} rows)")
