"""Error pattern of the projection US = A0 V (plan stages) against float64 numpy: which pixel rows /
tiles / TMEM quadrants / rank columns are wrong, over several repeats (race hunting)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle.fkk_oracle as O  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
I, R, _ = generate_rows(cfg, 0, n)
A = O.log_ratio(I, R, O.Params())
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, n, in_dtype=cfg.dtype)
Id, Rd = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
for rep in range(4):
    plan.transform(Id, Rd)
    V, US = plan.stage("V"), plan.stage("US")
    ref = A @ V
    err = np.abs(US - ref) / np.max(np.abs(ref))
    bad = err > 1e-5
    print(f"rep {rep}: max err {err.max():.3e}, bad entries {bad.sum()} of {bad.size}")
    if bad.any():
        rows, cols = np.nonzero(bad)
        tiles = np.unique(rows // 128)
        print("  tiles:", tiles[:20], "count", len(tiles), " CTA (tile % 148):", np.unique(tiles % 148)[:20])
        print("  rows within tile:", np.unique(rows % 128)[:40], " quadrants", np.unique((rows % 128) // 32))
        print("  rank columns:", np.unique(cols)[:64])
        t0 = tiles[0]
        e_t = err[t0 * 128:(t0 + 1) * 128]
        print("  first bad tile", t0, "max err per quadrant", [float(e_t[q * 32:(q + 1) * 32].max()) for q in range(4)])
