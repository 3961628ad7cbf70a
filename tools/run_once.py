"""One fKK-EC transform (cfg2 by default) and one direct-KK batch through the C-ABI: a short
command for `ncu --set full` captures of single kernels (tools/gpu_ncu_full.sh)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--direct-rows", type=int, default=8192)
ap.add_argument("--gemm", default=None)
a = ap.parse_args()
cfg = CONFIGS[a.workload]
n = a.rows or cfg.n_pixels
I, R, _ = generate_rows(cfg, 0, n)
Id, Rd = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, n, gemm=a.gemm, in_dtype=cfg.dtype)
K = plan.transform(Id, Rd)
if a.direct_rows:
    Kd = plan.direct(Id[: a.direct_rows], Rd)
torch.cuda.synchronize()
print("ok", float(K.imag.abs().max()))
