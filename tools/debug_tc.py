"""Probe the UMMA layouts: one tcgen05.mma per mode vs numpy."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402

rng = np.random.default_rng(0)
for N in (256, 64):
    A = rng.integers(-4, 5, (128, 8)).astype(np.float32)
    B = rng.integers(-4, 5, (N, 8)).astype(np.float32)
    ref = A @ B.T
    for mode in range(8):
        D = fkk.fkk_debug_tc_mma(mode, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
        err = np.abs(D - ref).max()
        extra = ""
        if err > 0:
            extra = f" nz={int((D != 0).sum())} D[0,:4]={D[0, :4]} ref[0,:4]={ref[0, :4]} D[1,:4]={D[1,:4]}"
        print(f"N={N} mode={mode} a_mn={mode & 1} b_mn={(mode >> 1) & 1} pad={(mode >> 2) & 1} maxerr={err}{extra}")
