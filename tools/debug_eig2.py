import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
from oracle import fkk_oracle as O
from synth import CONFIGS, generate_rows
cfg = CONFIGS["cfg2"]
I, R, _ = generate_rows(cfg, 0, 20000)
G = O.gram(O.log_ratio(I.astype(np.float64), R.astype(np.float64), O.Params()))
k = 40
ref = np.linalg.eigvalsh(G)[::-1]
def run(Gm, tag):
    V, lam = fkk.fkk_debug_eig_topk(torch.from_numpy(np.ascontiguousarray(Gm)).cuda(), k)
    V, lam = V.cpu().numpy(), lam.cpu().numpy()
    r = np.linalg.eigvalsh(Gm)[::-1][:k]
    print(tag, "lam err", np.max(np.abs(lam - r)) / r[0], "Vfin", np.isfinite(V).all(),
          "res", np.max(np.abs(Gm @ V - V * lam)) / r[0] if np.isfinite(V).all() else None)
run(G, "realG")
run(G / G.max(), "realG scaled")
rng = np.random.default_rng(0)
Q, _ = np.linalg.qr(rng.standard_normal((1000, 1000)))
run((Q * np.maximum(ref, 0)) @ Q.T, "same spectrum random vecs")
Gp = G.copy(); Gp += np.diag(rng.uniform(0, 1e-3, 1000)) * ref[0]
run(Gp, "realG + diag")
for M in (256, 512, 1000):
    run(G[:M, :M], f"realG[:{M}]")
