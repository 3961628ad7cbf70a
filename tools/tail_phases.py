"""Phase clocks of the cluster tail of the tridiagonalisation (FKK_TRIDIAG_DBG=13: rank 0, column M-100)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FKK_TRIDIAG_DBG"] = sys.argv[1] if len(sys.argv) > 1 else "13"
from paper_2005_07132_b200 import fkk
M = 1000
rng = np.random.default_rng(0)
Q, _ = np.linalg.qr(rng.standard_normal((M, M)))
G = torch.from_numpy((Q * np.linspace(1, 2, M)) @ Q.T).cuda()
for _ in range(50):
    d, e, t = fkk.fkk_debug_tridiag(G)
ts = d.cpu().numpy()[:5]
for i, nm in enumerate(["chain", "sync", "pass+push", "cluster barrier"]):
    print(f"{nm:16s} {ts[i + 1] - ts[i]:8.0f} cycles")
