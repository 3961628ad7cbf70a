"""Median per-stage times (plan CUDA events) of repeated fKK-EC transforms on a row block of a
BASELINE config (A/B of kernel variants selected by environment variables in separate processes).
   python tools/time_stages.py [cfg3|cfg4] [rows] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = CONFIGS[name]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_pixels
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 7
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True)
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
plan.transform(I, R, out)
st = []
for _ in range(reps):
    plan.transform(I, R, out)
    torch.cuda.synchronize()
    st.append(plan.stage_times())
med = {k: float(np.median([s[k] for s in st])) for k in st[0]}
env = {k: v for k, v in os.environ.items() if k.startswith("FKK_")}
print(json.dumps({"cfg": name, "rows": rows, "k": cfg.rank_k, "M": cfg.n_freq, "env": env,
                  "stage_ms_median": med, "total_ms": sum(med.values())}))
