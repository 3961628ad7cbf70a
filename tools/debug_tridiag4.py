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
d0, e0, t0 = [x.cpu().numpy() for x in fkk.fkk_debug_tridiag(G)]
chk("before")
big = torch.empty(int(3e8) // 4, dtype=torch.float32, device="cuda")
chk("after 300MB alloc")
del big
cfg = CONFIGS["cfg2"]
N = 20000
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, N)
I, R, _ = generate_rows(cfg, 0, N)
plan.svd(torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda())
chk("after svd")
d1, e1, t1 = [x.cpu().numpy() for x in fkk.fkk_debug_tridiag(G)]
print("tridiag diff after svd", np.max(np.abs(d1 - d0)), np.max(np.abs(e1[:-1] - e0[:-1])), np.max(np.abs(t1[:-2] - t0[:-2])))
print("G unchanged", np.array_equal(G.cpu().numpy(), Gn))
chk("again")
