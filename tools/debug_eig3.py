import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
from synth import CONFIGS, generate_rows
cfg = CONFIGS["cfg2"]
I, R, _ = generate_rows(cfg, 0, cfg.n_pixels)
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, cfg.n_pixels)
try:
    plan.svd(torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda())
except Exception as ex:
    print("svd failed", ex)
G = plan.stage("G")
np.save("gpurun_out/G_cfg2.npy", G)
k = 40
def run(Gm, tag):
    V, lam = fkk.fkk_debug_eig_topk(torch.from_numpy(np.ascontiguousarray(Gm)).cuda(), k)
    V, lam = V.cpu().numpy(), lam.cpu().numpy()
    r = np.linalg.eigvalsh(Gm)[::-1][:k]
    print(tag, "lam err", np.max(np.abs(lam - r)) / r[0], "Vfin", np.isfinite(V).all())
run(G, "gpuG")
run(G.copy(), "gpuG copy")
