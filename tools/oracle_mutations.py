"""Mutation sweep of the fp64 oracle: apply one plausible mistake at a time to a scratch copy of
oracle/fkk_oracle.py and check that tests/test_oracle_pins.py catches it.  A mutation that survives
marks an unpinned step (DESIGN.md section 2 lists the two survivors and why they are harmless).

    python tools/oracle_mutations.py            # ~3 min on 8 cores
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    # direct path D4 / D5 (Eq. 5, reading A9)
    "pec_sign": ("a2 = a + hilbert(phi_err, p)\n    phi2 = phi - phi_err",
                 "a2 = a - hilbert(phi_err, p)\n    phi2 = phi + phi_err"),
    "pec_amp_only": ("a2 = a + hilbert(phi_err, p)", "a2 = a"),
    "pec_phase_only": ("phi2 = phi - phi_err", "phi2 = phi"),
    "sec_mean": ("T = sg_trend(K1.real, sg_window(a.shape[1], p), p.sg_order)",
                 "T = K1.real.mean(axis=1, keepdims=True) * np.ones_like(K1.real)"),
    "sec_fallback_never": ("bad = T.min(axis=1) <= 0", "bad = T.min(axis=1) < -1e300"),
    # fPEC ridge (Eq. 17, reading A11)
    "ridge_trace": ("lam = p.ridge_rel * lambda_max_sym(C)", "lam = p.ridge_rel * np.trace(C)"),
    "ridge_zero": ("lam = p.ridge_rel * lambda_max_sym(C)", "lam = 0.0 * lambda_max_sym(C)"),
    # ALS (reading A6)
    "als_w_swap": ("w = np.where(yn > z, p.als_p, 1.0 - p.als_p)", "w = np.where(yn > z, 1.0 - p.als_p, p.als_p)"),
    "als_tie": ("w = np.where(yn > z, p.als_p, 1.0 - p.als_p)", "w = np.where(yn >= z, p.als_p, 1.0 - p.als_p)"),
    "als_iters_minus": ("for _ in range(p.als_iters):", "for _ in range(p.als_iters - 1):"),
    # SG trend (reading A8)
    "sgwin": ("return p.sg_window if p.sg_window else 2 * int(np.floor(0.375 * M)) + 1",
              "return p.sg_window if p.sg_window else 2 * int(np.floor(0.3 * M)) + 1"),
    "sg_edge": ("out[:, :h] = (Ve[:h] @ coef_lo).T", "out[:, :h] = y2[:, :h]"),
    # Hilbert (readings A2-A4)
    "hil_sign": ("h[1:L // 2] = -1j\n    h[L // 2 + 1:] = 1j", "h[1:L // 2] = 1j\n    h[L // 2 + 1:] = -1j"),
    "hil_nyq": ("h[L // 2 + 1:] = 1j", "h[L // 2:] = 1j"),
    "pad_pl": ("pl = (L - M) // 2\n    pr = L - M - pl\n    if p.pad", "pl = (L - M) // 2 + 1\n    pr = L - M - pl\n    if p.pad"),
    # log-ratio / noise scale (Eqs. 6, 9, 10; reading A16)
    "logratio_half": ("a = 0.5 * np.log(np.maximum(r, p.ratio_floor))", "a = np.log(np.maximum(r, p.ratio_floor))"),
    "floor": ("a = 0.5 * np.log(np.maximum(r, p.ratio_floor))", "a = 0.5 * np.log(np.maximum(r, 1e-3))"),
    "f_eq9": ("return 2.0 * mean / np.sqrt(p.f_alpha * mean + p.f_sigma_g ** 2)",
              "return 2.0 * mean / np.sqrt(p.f_alpha * mean + p.f_sigma_g)"),
    "f_apply_div": ("a = a * f[None, :]", "a = a / f[None, :]"),
    "vt_f_mul": ("Vt_f = V.T / f[None, :]", "Vt_f = V.T * f[None, :]"),
    # factorized path (Eqs. 13-23)
    "bamp_sign": ("B_amp = Vt_f + HPhi - v_sec", "B_amp = Vt_f - HPhi - v_sec"),
    "bph_sign": ("B_ph = Hv - phi_pec", "B_ph = Hv + phi_pec"),
    "vsec_noHPhi": ("v_sec = sg_trend(Vt_f + HPhi,", "v_sec = sg_trend(Vt_f,"),
    "q_argmax_only": ("return np.unique(np.concatenate([qmax, qmin]))", "return np.unique(qmax)"),
    "sign_rule": ("if V[j, i] < 0:", "if V[j, i] > 0:"),
    "eig_order": ("order = np.argsort(lam)[::-1]", "order = np.argsort(lam)"),
    "fpec_P": ("P = X @ Hv\n", "P = X @ (Hv * 0.5)\n"),
    "recon_conj": ("return np.exp(US @ B_amp) * np.exp(1j * (US @ B_ph))",
                   "return np.exp(US @ B_amp) * np.exp(-1j * (US @ B_ph))"),
    "ml_w": ("return V * (s ** 2 / (s ** 2 + lam))[None, :]", "return V * (s / (s ** 2 + lam))[None, :]"),
    "denoise": ("return (I @ V) @ V.T", "return (I @ V) @ V.T * 1.0001"),
    # randomized range finder
    "rr_no_power": ("for _ in range(q):", "for _ in range(0):"),
    "rr_no_reorth": ("Q = _orth(A.T @ Q)", "Q = A.T @ Q"),
}


def main():
    survivors = []
    src = open(os.path.join(ROOT, "oracle", "fkk_oracle.py")).read()
    for name, (old, new) in MUTATIONS.items():
        if old not in src:
            print(f"{name:20s} -> (pattern not found, skipped)")
            continue
        with tempfile.TemporaryDirectory() as d:
            for sub in ("oracle", "synth", "tests"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub))
            open(os.path.join(d, "oracle", "fkk_oracle.py"), "w").write(src.replace(old, new, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x", "-m", "not gpu",
                                "-p", "no:cacheprovider"], cwd=d, capture_output=True, text=True, timeout=1800)
            tail = [l for l in r.stdout.splitlines() if "passed" in l or "failed" in l]
            caught = r.returncode != 0
            print(f"{name:20s} -> {'caught' if caught else 'SURVIVED'}  ({tail[-1] if tail else '?'})", flush=True)
            if not caught:
                survivors.append(name)
    print("survivors:", survivors)


if __name__ == "__main__":
    main()
