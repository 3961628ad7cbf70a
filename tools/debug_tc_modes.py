import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk
rng = np.random.default_rng(0)
A = rng.standard_normal((128, 8)).astype(np.float32)
B = rng.standard_normal((64, 8)).astype(np.float32)
def tf(x):
    u = x.view(np.uint32).copy(); u = (u + 0x1000) & 0xffffe000; return u.view(np.float32).astype(np.float64)
ref = tf(A) @ tf(B).T
for mode in range(8):
    D = fkk.fkk_debug_tc_mma(mode, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    print(mode, np.max(np.abs(D - ref)), np.max(np.abs(ref)))
