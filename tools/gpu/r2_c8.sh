# direct_finish with 8 channels per thread at M = 1600 (float4 path): parity subset + cfg4-geometry direct timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "direct or conventional or paper or clamp or wide" > gpurun_out/c8_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/c8_tests.log
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2005_07132_b200 import fkk
from synth import CONFIGS, generate_rows
cfg = CONFIGS["cfg4"]; rows = 262144
I, R, _ = generate_rows(cfg, 0, rows)
I, R = torch.from_numpy(I).cuda(), torch.from_numpy(R).cuda()
out = torch.empty((rows, cfg.n_freq), dtype=torch.complex64, device="cuda")
plan = fkk.Plan(cfg.n_freq, cfg.rank_k, rows, timing=True)
plan.direct(I, R, out); torch.cuda.synchronize()
for _ in range(2):
    plan.direct(I, R, out); torch.cuda.synchronize()
    print("cfg4 geometry direct, 262144 rows:", plan.stage_times())
PY
timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn | tail -1
