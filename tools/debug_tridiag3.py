import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
from synth import CONFIGS, generate_rows
Gn = np.load("dbg/G_cfg2.npy")
G = torch.from_numpy(Gn).cuda()
ref = np.linalg.eigvalsh(Gn)[::-1]
def chk(tag):
    V, lam = fkk.fkk_debug_eig_topk(G, 40)
    print(tag, np.max(np.abs(lam.cpu().numpy() - ref[:40])) / ref[0], np.isfinite(V.cpu().numpy()).all(), flush=True)
chk("before")
cfg = CONFIGS["cfg2"]
N = int(os.environ.get("NR", "1024"))
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, N)
chk("after plan create")
I, R, _ = generate_rows(cfg, 0, N)
try:
    plan.svd(torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda())
    print("svd ok")
except Exception as ex:
    print("svd failed", ex)
chk("after svd")
del plan
chk("after plan destroy")
