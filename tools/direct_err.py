"""Max relative error of the direct path against the oracle on a cfg2 sample (numerics check)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402
import oracle.fkk_oracle as O  # noqa: E402
cfg = CONFIGS["cfg2"]
I, R, _ = generate_rows(cfg, 0, 300)
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, 300)
K = plan.direct(torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()).cpu().numpy()
Ko = O.kk_direct(I.astype(np.float64), R.astype(np.float64))
print("direct max rel err (row-wise max-norm):", np.max(np.max(np.abs(K - Ko), axis=1) / np.max(np.abs(Ko), axis=1)))
