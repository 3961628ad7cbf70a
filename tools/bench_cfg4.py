"""BASELINE.json configs[3] (cfg4: 4,000,000 x 1600, k = 100) on ONE B200: the full fKK-EC transform
(device-resident cube, CUDA events, 1 warm-up + 3 timed) and one direct-KK pass, with the stage split.
The cube is generated in 500,000-row blocks (synth.generate_rows, bit-identical to the whole-cube
generator) and copied into one device buffer (25.6 GB); the complex64 output is 51.2 GB.

    python tools/bench_cfg4.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2005_07132_b200 import fkk  # noqa: E402
from synth import CONFIGS, generate_rows  # noqa: E402


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "cfg4.json")
    cfg = CONFIGS["cfg4"]
    N, M, k = cfg.n_pixels, cfg.n_freq, cfg.rank_k
    t0 = time.time()
    I = torch.empty((N, M), dtype=torch.float32, device="cuda")
    Iref = None
    for r0 in range(0, N, 500_000):
        r1 = min(N, r0 + 500_000)
        Ib, Rb, _ = generate_rows(cfg, r0, r1)
        I[r0:r1].copy_(torch.from_numpy(Ib))
        Iref = Rb
    Iref = torch.from_numpy(Iref).cuda()
    gen_s = time.time() - t0
    out = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    plan = fkk.Plan(M, k, N, timing=True)
    plan.transform(I, Iref, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, acc = 3, {}
    e0.record()
    for _ in range(reps):
        plan.transform(I, Iref, out)
        for kk, v in plan.stage_times().items():
            acc[kk] = acc.get(kk, 0.0) + v / reps
    e1.record()
    torch.cuda.synchronize()
    t_f = e0.elapsed_time(e1) / reps
    g_ms = acc.get("gram", float("nan"))
    gram_tfs = N * M * M / (g_ms / 1e3) / 1e12
    plan.direct(I, Iref, out)
    plan.als_solves()
    torch.cuda.synchronize()
    e0.record()
    plan.direct(I, Iref, out)
    e1.record()
    torch.cuda.synchronize()
    t_d = e0.elapsed_time(e1)
    doc = {"workload": "cfg4 (BASELINE.json configs[3]): 4,000,000 x 1600, k = 100, fp32 cube, complex64 out, one B200",
           "fkk_ec": {"ms_per_pass": t_f, "spectra_per_s": N / (t_f / 1e3), "stage_ms": acc,
                      "gram_tflops_fp32_equiv": gram_tfs},
           "direct_kk": {"ms_per_pass": t_d, "spectra_per_s": N / (t_d / 1e3), "stage_ms": plan.stage_times(),
                         "als_solves_per_spectrum": plan.als_solves() / N},
           "generation_s": gen_s}
    print(json.dumps(doc))
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    json.dump(doc, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
