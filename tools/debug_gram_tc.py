"""Debug: Gram from the tcgen05 kernel vs fp64, saved to gpurun_out/gram_tc_debug.npz."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402

rng = np.random.default_rng(0)
N, M = int(sys.argv[1]) if len(sys.argv) > 1 else 256, int(sys.argv[2]) if len(sys.argv) > 2 else 512
a = rng.standard_normal((N, M)) * 0.1
Iref = np.ones(M, np.float32)
I = np.exp(2 * a).astype(np.float32)
A = 0.5 * np.log(I.astype(np.float64))
out = {}
for g in ["fp32_simt", "3xtf32"]:
    plan = fkk.Plan(M, 4, N, gemm=g)
    try:
        plan.svd(torch.from_numpy(I).cuda(), torch.from_numpy(Iref).cuda())
    except Exception as e:
        print(g, "svd error", e)
    out[g] = plan.stage("G")
G = A.T @ A
out["ref"] = G
np.savez("gpurun_out/gram_tc_debug.npz", **out)
for g in ["fp32_simt", "3xtf32"]:
    d = out[g]
    print(g, "nan", np.isnan(d).sum(), "maxrel", np.nanmax(np.abs(d - G)) / np.abs(G).max(),
          "zeros", (d == 0).sum(), "diag ratio", np.nanmedian(np.diag(d) / np.diag(G)))
