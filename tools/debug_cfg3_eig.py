"""Diagnose the eigensolver on the cfg3 Gram (GPU G from fkk_svd stage dump vs numpy eigh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_pixels
I, R, _ = generate_rows(cfg, 0, n)
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, n)
Id, Rd = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
try:
    plan.transform(Id, Rd)
    print("transform ok")
except Exception as ex:  # noqa: BLE001
    print("transform failed:", ex)
G = plan.stage("G")
print("G finite", np.isfinite(G).all(), "sym", np.max(np.abs(G - G.T)))
k = cfg.rank_k
V, lam = fkk.fkk_debug_eig_topk(torch.from_numpy(G).cuda(), k)
V, lam = V.cpu().numpy(), lam.cpu().numpy()
ref = np.linalg.eigvalsh(G)[::-1]
print("lam finite", np.isfinite(lam).all(), "V finite", np.isfinite(V).all())
print("lam err", np.max(np.abs(lam - ref[:k])) / ref[0])
print("res", np.max(np.abs(G @ V - V * lam)) / ref[0], "orth", np.max(np.abs(V.T @ V - np.eye(k))))
print("top eigs", ref[:5], "k-th", ref[k - 1], ref[k])
