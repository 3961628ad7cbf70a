import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
Gn = np.load("dbg/G_cfg2.npy")
G = torch.from_numpy(Gn).cuda()
ref = np.linalg.eigvalsh(Gn)[::-1]
for force in ("0", "1"):
    os.environ["FKK_EIG_FORCE_L2"] = force
    for k in (1, 2, 8, 40):
        V, lam = fkk.fkk_debug_eig_topk(G, k)
        lam = lam.cpu().numpy(); V = V.cpu().numpy()
        print(force, k, lam[:3], ref[:3], "Vfin", np.isfinite(V).all(), np.isfinite(V).sum(axis=0)[:4])
