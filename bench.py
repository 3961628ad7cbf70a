"""bench.py -- throughput of the fKK-EC hot path on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg3]

A step is one pass of the hot path over the configuration-3 image (703,026 spectra x 1,000
channels, k = 60; BASELINE.json configs[2]): the full factorized fKK-EC transform F0..F11 through
the C-ABI (fkk_transform) on device-resident inputs.  `value` = spectra/s of that transform, whole
job (N GPUs shard the pixels of the same image: strong scaling).  In the same run the two other hot
paths are timed and reported as sub-objects: the direct per-spectrum KK+PEC+SEC (kk_direct_batch)
on the same image, and ML:fKK-EC apply (fkk_apply_trained_basis, BASELINE.json configs[4]).

Multi-GPU: launched by torchrun, one rank per GPU; NCCL unique id bootstrap through
torch.distributed; barrier + max over ranks of the device-timed step.
The oracle (oracle/, test infrastructure) is executed only in the cpu_baseline leg (rank 0,
N=1) and in --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch of the hot kernels, extracted
# from a committed capture by tools/ncu_traffic.py (profiles/*_traffic.json); labelled with its source
def _traffic():
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return {}, None
    try:
        return json.load(open(files[-1])), os.path.relpath(files[-1], ROOT)
    except Exception:
        return {}, None


METRIC = "spectra/s for full fKK-EC (and direct KK) at 1/2/4/8 B200; % HBM/TC roofline"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows: list[list[str]] = []
        self.proc = None
        self.start = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a few hundred ms to emit its first row; a 0.2 s timed region could end
            # before it (one run came back "unsampled"): wait for the sampler to be live, then count
            # only the rows that arrive from here on (the timed region)
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.start = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[self.start:] or self.rows[-1:]   # (a region shorter than one 20 ms period: the last row)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.rows = rows
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world: int):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def run_ours(args) -> dict:
    import torch

    from paper_2005_07132_b200 import fkk
    from synth import CONFIGS, generate_rows

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [fkk.fkk_get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    cfg = CONFIGS[args.workload]
    N, M, k = cfg.n_pixels, cfg.n_freq, cfg.rank_k
    r0, r1 = fkk.fkk_shard_range(N, world, rank)
    n_loc = r1 - r0
    I_h, Iref_h, _ = generate_rows(cfg, r0, r1)
    I = torch.from_numpy(I_h).cuda()
    Iref = torch.from_numpy(Iref_h).cuda()
    out = torch.empty((n_loc, M), dtype=torch.complex64, device="cuda")
    plan = fkk.Plan(M, k, n_loc, timing=True, world_size=world, rank=rank, nccl_id=nccl_id, device=local)
    stream = torch.cuda.current_stream()

    # ---------------- fKK-EC (the headline) ----------------
    for _ in range(args.warmup):
        plan.transform(I, Iref, out)
    _barrier(world)
    stage_acc: dict = {}
    launches = 0
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        _barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            plan.transform(I, Iref, out)
            for kk, v in plan.stage_times().items():
                stage_acc[kk] = stage_acc.get(kk, 0.0) + v
            launches += plan.launches
        ev1.record(stream)
        _barrier(world)
    t_loc = ev0.elapsed_time(ev1) / args.steps
    t = _max_over_ranks(t_loc, world)
    stage_ms = {kk: v / args.steps for kk, v in stage_acc.items()}
    value = N / (t / 1e3)

    # per-run parity diagnostics of the last timed transform (outside the timed region):
    # the eigengap at k and the GPU eigenvalues against a host fp64 eigvalsh of the same G, the
    # argmax/argmin margins of the US columns that decide q, the size of q, clamped / non-finite inputs
    diag = None
    if world == 1:
        G_h = plan.stage("G")
        lam_h = np.linalg.eigvalsh(G_h)[::-1]
        s_gpu = plan.stage("S")[:k]
        s_h = np.sqrt(np.maximum(lam_h[:k], 0.0))
        US_h = plan.stage("US")[:n_loc, :k]
        two = np.partition(US_h, [n_loc - 2, n_loc - 1], axis=0)[-2:]      # 2nd largest, largest
        low = np.partition(US_h, [0, 1], axis=0)[:2]                        # smallest, 2nd smallest
        scale = np.max(np.abs(US_h), axis=0)
        diag = {"eigengap_k_rel": float((lam_h[k - 1] - lam_h[k]) / lam_h[k - 1]),
                "sigma_k_over_sigma_1": float(s_h[k - 1] / s_h[0]),
                "max_abs_ds_over_s1_gpu_vs_host_eigvalsh": float(np.max(np.abs(s_gpu - s_h)) / s_h[0]),
                "argmax_margin_min_rel": float(np.min((two[1] - two[0]) / scale)),
                "argmin_margin_min_rel": float(np.min((low[1] - low[0]) / scale)),
                "n_q": int(plan.stage("Q").size),
                "clamped_inputs": int(np.count_nonzero(I_h < 1e-6 * Iref_h[None, :])),
                "nonfinite_inputs": int(np.count_nonzero(~np.isfinite(I_h)))}
        del G_h, US_h

    # roofline of the Gram (F2, tcgen05 3xTF32): algorithmic flops N*M^2 (the syrk: M(M+1)/2 unique
    # products x 2 flops, rounded to M^2) per pass; 3xTF32 issues three TF32 products per fp32-equivalent
    # product, so its fp32-equivalent peak is the TF32 peak / 3.  The denominator is
    # the BURST bf16 figure (scaled by the guide's nominal TF32/BF16 ratio) unless this run's clock record
    # shows the power cap, in which case it is the sustained one (B200_PROFILING.md).
    peaks, src = _peaks()
    clocks = clk.summary()
    capped = "sw_power_cap" in clocks.get("reasons", [])
    traffic, traffic_src = _traffic()
    gram_ms = stage_ms.get("gram", float("nan"))
    gram_flops = float(n_loc) * M * M
    bf16 = peaks["bf16_tflops_sustained"] if capped else peaks["bf16_tflops"]
    peak_3x = bf16 * (1.1 / 2.25) / 3.0
    achieved = gram_flops / (gram_ms / 1e3) / 1e12
    pair = ((M + 127) // 128) % 2 == 0
    gname = "gram_pre2" if pair else "gram_pre"
    tr = traffic.get(args.workload, {}).get(gname)
    roofline = {"kernel": (f"{gname} (F2, tcgen05.mma {'cta_group::2 ' if pair else ''}kind::tf32 "
                           f"{'256x256' if pair else '128x128'} tiles, 3xTF32 from the pre-split A0 image)"),
                "bound": "tensor", "achieved": achieved, "peak": peak_3x, "unit": "TFLOP/s", "frac": achieved / peak_3x,
                "traffic": tr,
                "traffic_source": (f"ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch, {traffic_src}"
                                   if tr else "not captured for this workload"),
                "peak_source": (f"{src} {'sustained' if capped else 'burst'} bf16 {bf16:.0f} TF/s x 1.1/2.25 (nominal "
                                f"TF32/BF16) / 3 (3xTF32 products); {'sw_power_cap seen' if capped else 'no power cap seen'} "
                                f"during the timed region; algorithmic flops = N*M^2 per pass; CUDA events on the plan "
                                f"stream (the Gram kernel + its fp64 split reduction)")}
    # per-kernel rooflines of the other hot kernels (same event timing)
    hbm = peaks["hbm_gbs"]
    other = {}
    # logratio_pre reads the cube and writes the tf32 hi/lo MMA image of A0 for the Gram (128-channel
    # blocks x 32-pixel stages of 2 x 16,640 B); A0 itself is not stored: the projection reads the cube
    # again and forms A0 in its converter warps
    image_bytes = 2.0 * ((M + 127) // 128) * ((n_loc + 31) // 32) * 16640
    for name, nbytes in (("logratio", 4.0 * n_loc * M + image_bytes), ("project", 4.0 * n_loc * M + 4.0 * n_loc * k),
                         ("reconstruct", 8.0 * n_loc * M + 4.0 * n_loc * k)):
        ms = stage_ms.get(name)
        if ms:
            gbs = nbytes / (ms / 1e3) / 1e9
            other[name] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                           "bytes_per_pass": nbytes}
    roofline["others"] = other

    # ---------------- direct KK (same image) ----------------
    # timed on a plan without stage events (no event records between kernels); the per-stage split
    # comes from one more pass of the timing plan
    pdir = fkk.Plan(M, k, n_loc, device=local)
    pdir.direct(I, Iref, out)
    pdir.als_solves()
    _barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    nd = max(1, min(args.steps, 3))
    e0.record(stream)
    for _ in range(nd):
        pdir.direct(I, Iref, out)
    e1.record(stream)
    _barrier(world)
    td = _max_over_ranks(e0.elapsed_time(e1) / nd, world)
    solves = pdir.als_solves() / (nd * n_loc)
    del pdir
    plan.direct(I, Iref, out)          # (the plan's first direct call allocates its phi / phi_err scratch)
    plan.direct(I, Iref, out)
    dstage = plan.stage_times()
    # rooflines of the direct path: ALS against the FP64 pipe (algorithmic flops
    # = 25 M per solve: the serial pentadiagonal LDL^T + forward + back substitution, times the solves
    # actually needed); the two Hilbert kernels against FP32 (5 L log2 L flops per complex transform,
    # two transforms per spectrum pair and Hilbert) and HBM (bytes they must move)
    fp64_peak = 37.2e12    # measured DFMA throughput (tools/micro/lat.cu): 148 SM x 64 x 2 x 1.965 GHz
    fp32_peak = 148 * 128 * 2 * 1.965e9
    L = 2 * (1 << (M - 1).bit_length())
    hil_fl = 5.0 * L * np.log2(L)              # per spectrum (two-for-one) and Hilbert round trip
    dr = {}
    if dstage.get("als"):
        fl = 25.0 * M * solves * n_loc
        a = fl / (dstage["als"] / 1e3)
        dr["als"] = {"bound": "fp64", "achieved": a / 1e12, "peak": fp64_peak / 1e12, "unit": "TFLOP/s",
                     "frac": a / fp64_peak, "solves_per_spectrum": solves,
                     "flops_per_spectrum": 25.0 * M * solves}
    for nm, fl_s, by_s in (("kk_phase", hil_fl, 8.0 * M), ("pec_sec", hil_fl + 40.0 * M, 20.0 * M)):
        ms = dstage.get(nm)
        if ms:
            a_fl = fl_s * n_loc / (ms / 1e3)
            a_by = by_s * n_loc / (ms / 1e3)
            dr[nm] = {"bound": "fp32 (FFT)", "achieved": a_fl / 1e12, "peak": fp32_peak / 1e12, "unit": "TFLOP/s",
                      "frac": a_fl / fp32_peak, "hbm_gbs": a_by / 1e9, "hbm_frac": a_by / (hbm * 1e9)}
    direct_kk = {"value": N / (td / 1e3), "unit": "spectra/s", "ms_per_pass": td,
                 "stage_ms": dstage, "stage_sum_ms": sum(dstage.values()),
                 "als_solves_per_spectrum": solves, "roofline": dr}

    # ---------------- randomized range finder in place of Gram + eigensolver -------
    # timed at q = args.rf_q power iterations; accuracy against this run's Gram path at q = 1, 2, 4, 8
    rfo = None
    if not args.skip_ml:
        plan.transform(I, Iref, out)
        s_g, V_g, q_g = plan.stage("S"), plan.stage("V"), plan.stage("Q")
        samp = torch.arange(0, n_loc, 97, device=out.device)
        kg = out[samp].imag.clone()
        out_rf = torch.empty_like(out)
        acc = {}
        for qi in sorted({args.rf_q, 1, 2, 4, 8}):
            prf = fkk.Plan(M, k, n_loc, timing=True, world_size=world, rank=rank, nccl_id=nccl_id, device=local,
                           svd="range_finder", rf_oversample=10, rf_power_iters=qi)
            prf.transform(I, Iref, out_rf)
            _barrier(world)
            nr = max(1, min(args.steps, 5)) if qi == args.rf_q else 1
            racc: dict = {}
            e0.record(stream)
            for _ in range(nr):
                prf.transform(I, Iref, out_rf)
                for kk, v in prf.stage_times().items():
                    racc[kk] = racc.get(kk, 0.0) + v / nr
            e1.record(stream)
            _barrier(world)
            trf = _max_over_ranks(e0.elapsed_time(e1) / nr, world)
            s_r, V_r = prf.stage("S"), prf.stage("V")
            cos = np.linalg.svd(V_g.T @ V_r, compute_uv=False)
            kr = out_rf[samp].imag
            acc[qi] = {"ms_per_pass": trf, "max_ds_over_s1": float(np.max(np.abs(s_r - s_g)) / s_g[0]),
                       "min_principal_cosine": float(cos.min()),
                       "same_q": bool(np.array_equal(q_g, prf.stage("Q"))),
                       "im_k_maxnorm_rel_diff_sampled": float((kr - kg).abs().max() / kg.abs().max())}
            if qi == args.rf_q:
                rfo = {"value": N / (trf / 1e3), "unit": "spectra/s", "ms_per_pass": trf, "stage_ms": racc,
                       "oversample": 10, "power_iters": qi}
            del prf
        rfo["accuracy_vs_gram_path_by_power_iters"] = acc
        del out_rf

    # ---------------- conventional workflow (Fig. 1(a): SVD denoise of the raw cube + direct KK) ----------
    conv = None
    if world == 1 and not args.skip_ml:
        k_keep = 6   # the paper's simulations kept 6 for the conventional workflow
        plan.conventional(I, Iref, k_keep, out)
        e0.record(stream)
        plan.conventional(I, Iref, k_keep, out)
        e1.record(stream)
        torch.cuda.synchronize()
        tc_ = e0.elapsed_time(e1)
        conv = {"value": N / (tc_ / 1e3), "unit": "spectra/s", "ms_per_pass": tc_, "k_keep": k_keep,
                "stage_ms": plan.stage_times()}

    # ---------------- ML:fKK-EC apply (config 5) ----------------
    ml = None
    if not args.skip_ml:
        tr = CONFIGS["cfg5_train"]
        ap = CONFIGS["cfg5_apply"]
        It_h, Rt_h, _ = generate_rows(tr, 0, tr.n_pixels)
        ptrain = fkk.Plan(tr.n_freq, tr.rank_k, tr.n_pixels, device=local)
        _, basis = ptrain.transform(torch.from_numpy(It_h).cuda(), torch.from_numpy(Rt_h).cuda(), return_basis=True)
        del ptrain
        a0, a1 = fkk.fkk_shard_range(ap.n_pixels, world, rank)
        Ia_h, _, _ = generate_rows(ap, a0, a1)
        Ia = torch.from_numpy(Ia_h).cuda()
        batch = 50000
        papply = fkk.Plan(ap.n_freq, ap.rank_k, batch, device=local)
        oa = torch.empty((batch, ap.n_freq), dtype=torch.complex64, device="cuda")
        for b0 in range(0, min(a1 - a0, batch), batch):
            papply.apply(basis, Ia[b0:b0 + batch], oa[: min(batch, a1 - a0 - b0)])
        _barrier(world)
        e0.record(stream)
        nb = 0
        for b0 in range(0, a1 - a0, batch):          # enqueued back to back (no host sync per batch)
            nbb = min(batch, a1 - a0 - b0)
            papply.apply(basis, Ia[b0:b0 + nbb], oa[:nbb])
            nb += 1
        e1.record(stream)
        _barrier(world)
        tm1 = _max_over_ranks(e0.elapsed_time(e1), world)
        # independent batches rotate over three streams (three plans, three output buffers): one batch's
        # projection fills the SMs the other's reconstruction tail leaves idle
        nst = int(os.environ.get("FKK_BENCH_ML_STREAMS", "3"))   # (A/B knob; 2 / 3 / 4: 0.1248 / 0.1225 / 0.1229 ms)
        plans2 = [papply] + [fkk.Plan(ap.n_freq, ap.rank_k, batch, device=local) for _ in range(nst - 1)]
        outs2 = [oa] + [torch.empty_like(oa) for _ in range(nst - 1)]
        sts = [torch.cuda.Stream(device=local) for _ in range(nst)]
        for b in range(nst):
            with torch.cuda.stream(sts[b]):
                plans2[b].apply(basis, Ia[:batch], outs2[b])
        torch.cuda.synchronize()
        _barrier(world)
        e0.record(stream)
        for st in sts:
            st.wait_event(e0)
        for i, b0 in enumerate(range(0, a1 - a0, batch)):
            nbb = min(batch, a1 - a0 - b0)
            with torch.cuda.stream(sts[i % nst]):
                plans2[i % nst].apply(basis, Ia[b0:b0 + nbb], outs2[i % nst][:nbb])
        for st in sts:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)
        e1.record(stream)
        _barrier(world)
        tm = _max_over_ranks(e0.elapsed_time(e1), world)
        del plans2[1:], outs2[1:]
        nbytes = 12.0 * (a1 - a0) * ap.n_freq           # read the cube (4 B) + write complex64 K (8 B) per element
        gbs = nbytes / (tm / 1e3) / 1e9
        ptime = fkk.Plan(ap.n_freq, ap.rank_k, batch, device=local, timing=True)   # per-kernel split of one full batch
        ptime.apply(basis, Ia[:batch], oa)
        ptime.apply(basis, Ia[:batch], oa)
        ml = {"value": ap.n_pixels / (tm / 1e3), "unit": "spectra/s", "ms_per_pass": tm,
              "batches": nb, "ms_per_batch": tm / max(nb, 1), "streams": nst, "ms_per_batch_one_stream": tm1 / max(nb, 1),
              "workload": "cfg5: apply 703,026 x 1000 (k=40) in 50,000-spectrum batches",
              "stage_ms_full_batch": ptime.stage_times(),
              "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                           "bytes_per_pass": nbytes}}
        del Ia, ptime
    else:
        papply = basis = Ia_h = batch = None

    # ---------------- end to end through the host-buffer C-ABI ----------------
    e2e = None
    if not args.skip_e2e:
        Ih = torch.from_numpy(I_h).pin_memory()
        Rh = torch.from_numpy(Iref_h).pin_memory()
        Oh = torch.empty((n_loc, M), dtype=torch.complex64).pin_memory()
        Oh2 = torch.empty((n_loc, M), dtype=torch.complex64).pin_memory()
        # one cube per call (context): H2D, transform, D2H in sequence
        plan.transform_host(Ih, Rh, Oh)
        _barrier(world)
        t0 = time.perf_counter()
        plan.transform_host(Ih, Rh, Oh)
        _barrier(world)
        t_single = _max_over_ranks(time.perf_counter() - t0, world)
        # the e2e number: consecutive cubes through fkk_transform_host_stream (cube i+1's H2D and cube
        # i-1's D2H overlap cube i's transform; each cube gets its full transform)
        plan.transform_host_stream([Ih, Ih], Rh, [Oh, Oh2])
        ne = max(2, min(args.steps, 8))
        _barrier(world)
        t0 = time.perf_counter()
        lat = plan.transform_host_stream([Ih] * ne, Rh, [Oh if i % 2 == 0 else Oh2 for i in range(ne)])
        _barrier(world)
        te = _max_over_ranks((time.perf_counter() - t0) / ne, world)
        e2e = {"value": N / te, "unit": "spectra/s", "h2d_bytes_per_step": int(I_h.nbytes + Iref_h.nbytes),
               "d2h_bytes_per_step": int(Oh.numel() * 8), "ms_per_step": te * 1e3, "cubes": ne,
               "cube_latency_ms_median": float(np.median(lat)),
               "how": "fkk_transform_host_stream: pinned host cube -> device, transform, complex64 cube -> pinned "
                      "host, per cube; the copies of neighbouring cubes overlap the transforms",
               "single_cube_call": {"value": N / t_single, "ms": t_single * 1e3, "how": "fkk_transform_host"}}
        del Oh2
        if ml is not None and world == 1 and Ia_h.shape == tuple(Ih.shape):
            # config 5 streamed from pinned host memory in 50,000-spectrum batches (H2D, apply, D2H pipelined)
            Ih.copy_(torch.from_numpy(Ia_h))
            papply.apply_stream(basis, Ih, Oh, batch)
            t0 = time.perf_counter()
            lat = papply.apply_stream(basis, Ih, Oh, batch)
            ts = time.perf_counter() - t0
            ml["e2e"] = {"value": Ia_h.shape[0] / ts, "unit": "spectra/s", "ms_per_pass": ts * 1e3,
                         "h2d_bytes_per_pass": int(Ia_h.nbytes), "d2h_bytes_per_pass": int(Oh.numel() * 8),
                         "batch_latency_ms": {"median": float(np.median(lat)), "max": float(np.max(lat)),
                                              "min": float(np.min(lat))},
                         "how": "fkk_apply_trained_basis_stream: pinned host cube, per batch H2D / apply / D2H on "
                                "three streams with two device buffer pairs"}

    res = {
        "metric": METRIC, "value": value, "unit": "spectra/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator synth/, BASELINE.json configs[2])",
        "config": {"workload": f"{args.workload}: fKK-EC transform of {N:,} x {M} (k={k}), fp32 cube, complex64 out",
                   "n_spectra": N, "n_freq": M, "rank_k": k, "parallelism": f"pixel shards x{world}",
                   "l2": "inputs larger than L2 (cube 2.81 GB, output 5.62 GB)"},
        "roofline": roofline, "stage_ms": stage_ms, "clocks": clocks, "parity_diagnostics": diag,
        "gpu_launches": int(launches),
        "direct_kk": direct_kk,
        "ml_apply": ml, "e2e": e2e, "conventional": conv, "range_finder": rfo,
    }
    return res


def cpu_baseline(args, kind="oracle", repeats: int = 3, n_s: int | None = None) -> dict:
    """The fp64 oracle as it stands, on the host cores, on a bounded sample of the same workload:
    mean +- std of `repeats` runs (the paper's protocol).  The inputs are generated
    once; the direct-KK oracle is timed once on its own (smaller) sample."""
    from oracle import fkk_oracle as O
    from synth import CONFIGS, generate_rows
    cfg = CONFIGS[args.workload]
    n_s = args.cpu_sample if n_s is None else n_s
    I, Iref, _ = generate_rows(cfg, 0, n_s)
    ts = []
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        O.fkk_ec(I, Iref, cfg.rank_k, O.Params())
        ts.append(time.perf_counter() - t0)
    dt = statistics.mean(ts)
    nd = min(args.cpu_direct_sample, n_s)
    t1 = time.perf_counter()
    O.kk_direct(I[:nd], Iref, O.Params())
    dd = time.perf_counter() - t1
    cores = len(os.sched_getaffinity(0))
    return {"value": n_s / dt, "unit": "spectra/s", "cores": cores, "kind": kind,
            "std": statistics.stdev([n_s / t for t in ts]) if len(ts) > 1 else 0.0, "repeats": len(ts),
            "step_values": [n_s / t for t in ts],
            "sample": f"fKK-EC oracle (fp64 NumPy, BLAS threads = {cores}) on the first {n_s:,} spectra of {args.workload}, "
                      f"mean of {len(ts)} runs ({dt:.1f} s each; the fixed eig/basis cost is amortised over the sample only); "
                      f"direct-KK oracle on {nd:,} spectra: {nd / dd:.1f} spectra/s",
            "direct_kk_value": nd / dd}


def run_reference(args) -> dict:
    """`--impl reference`: the oracle alone (this paper has no reference implementation).  Each step is one
    fKK-EC oracle pass over the same bounded sample (`--ref-sample` spectra, generated once); at most one
    warm-up pass, then exactly `--steps` timed passes; `value` = the median pass."""
    world, rank, local = _dist()
    if rank != 0:
        return {}
    n_s = args.ref_sample
    cb = cpu_baseline(args, kind="oracle", repeats=min(1, args.warmup) + max(1, args.steps), n_s=n_s)
    vals = cb.pop("step_values")[min(1, args.warmup):]
    v = statistics.median(vals)
    cb["value"] = v
    cb["repeats"] = len(vals)
    cb["std"] = statistics.stdev(vals) if len(vals) > 1 else 0.0
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "spectra/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n_s / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{args.workload} (bounded sample of {n_s:,} spectra per step)"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "spectra/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--cpu-sample", type=int, default=65536)
    ap.add_argument("--cpu-direct-sample", type=int, default=500)
    ap.add_argument("--ref-sample", type=int, default=16384,
                    help="spectra per step of the --impl reference arm (the oracle's fixed eig/basis cost is paid every step)")
    ap.add_argument("--skip-ml", action="store_true")
    ap.add_argument("--rf-q", type=int, default=1, help="power iterations of the range-finder sub-measurement")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, _ = _dist()
    if args.impl == "reference":
        res = run_reference(args)
        if rank == 0:
            print(json.dumps(res))
        return
    res = run_ours(args)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
