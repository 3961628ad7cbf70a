import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FKK_TRIDIAG_DBG"] = "3"
from paper_2005_07132_b200 import fkk
M = 1000
rng = np.random.default_rng(0)
Q, _ = np.linalg.qr(rng.standard_normal((M, M)))
G = torch.from_numpy((Q * np.linspace(1, 2, M)) @ Q.T).cuda()
for _ in range(200):
    d, e, t = fkk.fkk_debug_tridiag(G)
ts = e.cpu().numpy()[:8]
names = ["loads..w, x", "nrm", "v + sync", "pass", "bar syncthreads", "bar red+poll", "bar syncthreads"]
for i, nm in enumerate(names):
    print(f"{nm:14s} {ts[i + 1] - ts[i]:8.0f} cycles")
print("total", ts[7] - ts[0])
