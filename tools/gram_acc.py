"""Gram accuracy at scale: GPU G (default kernel) vs the fp64 oracle Gram on the first N cfg3 spectra."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fkk_oracle as O  # noqa: E402
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402

cfg = CONFIGS["cfg3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
I, R, _ = generate_rows(cfg, 0, n)
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, n)
plan.svd(torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda())
G = plan.stage("G")
Gor = O.gram(O.log_ratio(I.astype(np.float64), R.astype(np.float64), O.Params()))
print(f"N={n}: Gram max-norm relative error {np.max(np.abs(G - Gor)) / np.max(np.abs(Gor)):.3e}")
