"""Pins of the fp64 oracle against things other than itself (DESIGN.md "Oracle pins" P1..P20):
closed forms, brute force on tiny inputs, library routines for special cases, invariants, and
the values the paper/SPEC print (tests/golden/paper_values.json).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import fkk_oracle as O
from synth import CONFIGS, generate, lorentzian_spectrum, truth_imag

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
P0 = O.Params()
PN = O.Params(pad="none")
PZ = O.Params(pad="zero")


# ---------------------------------------------------------------- Hilbert ---------------------
def test_P1_hilbert_sign_periodic():
    L = 64
    n = np.arange(L)
    c = np.cos(2 * np.pi * 3 * n / L)
    s = np.sin(2 * np.pi * 3 * n / L)
    assert np.max(np.abs(O.hilbert(c, PN)[0] - s)) < 1e-13      # H{cos} = sin
    assert np.max(np.abs(O.hilbert(s, PN)[0] + c)) < 1e-13      # H{sin} = -cos


@pytest.mark.parametrize("L", [1024, 2048])
def test_P2_kk_exact_on_outer_function(L):
    """K(theta) = prod_j (1 - r_j e^{i(theta - theta_j)}) has no zeros in the unit disk, so ln K is
    a one-sided Fourier series and arg K = H{ln|K|} exactly; with I = |K|^2, I_ref = 1 the KK of
    Eq. 3 must return K itself."""
    rng = np.random.default_rng(1)
    th = 2 * np.pi * np.arange(L) / L
    K = np.ones(L, dtype=complex)
    for r in (0.9, 0.7, 0.5):
        K *= 1 - r * np.exp(1j * (th - rng.uniform(0, 2 * np.pi)))
    Kr = O.kk(np.abs(K)[None, :] ** 2, np.ones(L), PN)[0]
    assert np.max(np.abs(Kr - K)) / np.max(np.abs(K)) < 1e-12


def test_P3_constant_annihilated_reflect_only():
    for M in (512, 1000, 1600, 513):
        x = np.full((1, M), 3.7)
        assert np.max(np.abs(O.hilbert(x, P0))) < 1e-12
        assert np.max(np.abs(O.hilbert(x, PZ))) > 0.5       # zero padding: edge response


def test_P4_linearity():
    rng = np.random.default_rng(2)
    y, z = rng.standard_normal((2, 3, 700))
    a, b = 1.7, -0.3
    lhs = O.hilbert(a * y + b * z)
    rhs = a * O.hilbert(y) + b * O.hilbert(z)
    assert np.max(np.abs(lhs - rhs)) < 1e-12


def _reflect_index(i, M):
    period = 2 * (M - 1)
    j = i % period
    return j if j < M else period - j


@pytest.mark.parametrize("pad", ["reflect", "zero"])
@pytest.mark.parametrize("M", [40, 64, 37])
def test_P5_hilbert_brute_force(pad, M):
    """Direct O(L^2) sums: x_ext by the explicit reflection map, kernel g[j] = (2/L) sum_{k=1}^{L/2-1}
    sin(2 pi j k / L) (the impulse response of the -i sgn multiplier with DC/Nyquist zeroed)."""
    p = O.Params(pad=pad)
    L = O.fft_length(M, p)
    pl = (L - M) // 2
    rng = np.random.default_rng(M)
    x = rng.standard_normal(M)
    xe = np.zeros(L)
    for i in range(L):
        if pad == "reflect":
            xe[i] = x[_reflect_index(i - pl, M)]
        elif pl <= i < pl + M:
            xe[i] = x[i - pl]
    k = np.arange(1, L // 2)
    g = np.array([(2.0 / L) * np.sum(np.sin(2 * np.pi * j * k / L)) for j in range(L)])
    ref = np.array([sum(xe[n] * g[(m + pl - n) % L] for n in range(L)) for m in range(M)])
    assert np.max(np.abs(O.hilbert(x, p)[0] - ref)) < 1e-11


def test_P6_kk_single_lorentzian_matches_physics():
    gd = GOLD["lorentzian_kk_example"]
    w = np.linspace(500, 3800, 1000)
    chi = lorentzian_spectrum(w, gd["centre"], gd["hwhm"], gd["amp"], gd["chi_nr"])
    I = np.abs(chi) ** 2
    Iref = np.full(1000, gd["chi_nr"] ** 2)
    K = O.kk(I[None], Iref, P0)[0]
    truth = (chi / gd["chi_nr"]).imag
    j = int(np.argmin(np.abs(w - gd["centre"])))
    assert K.imag[j] > 0                                                # sign (A2)
    assert abs(truth[j] - gd["im_peak"]) / gd["im_peak"] < gd["rel_tol"]  # analytic peak ~ 0.2
    assert np.max(np.abs(K.imag - truth)) < gd["rel_tol"] * gd["im_peak"]


# ---------------------------------------------------------------- direct path -----------------
def test_P7_passthrough_zero_phase_error():
    """I = I_ref (K == 1) and I = c I_ref: PEC/SEC leave a zero-phase-error spectrum unchanged."""
    rng = np.random.default_rng(3)
    Iref = rng.uniform(0.5, 1.5, 512)
    for c in (1.0, 2.5):
        K = O.kk_direct((c * Iref)[None], Iref, P0)
        assert np.max(np.abs(K - 1.0)) < 1e-12


def test_P8_direct_scale_invariance():
    I, Iref, _ = generate(CONFIGS["cfg1"])
    rows = I[:6]
    K1 = O.kk_direct(rows, Iref, P0)
    K2 = O.kk_direct(3.0 * rows, Iref, P0)
    assert np.max(np.abs(K1 - K2)) / np.max(np.abs(K1)) < 1e-12


# ---------------------------------------------------------------- ALS -------------------------
def _als_dense(y, lam, p, iters):
    M = len(y)
    D = np.diff(np.eye(M), n=2, axis=0)
    w = np.ones(M)
    for _ in range(iters):
        z = np.linalg.solve(np.diag(w) + lam * D.T @ D, w * y)
        w = np.where(y > z, p, 1 - p)
    return z


def test_P9_als_line_shift_and_dense():
    M = 256
    t = np.arange(M, dtype=float)
    line = 0.3 - 0.002 * t
    z = O.als_baseline(line)[0]
    assert np.max(np.abs(z - line)) < 1e-7
    rng = np.random.default_rng(4)
    y = np.cumsum(rng.standard_normal(M)) * 0.05 + np.exp(-((t - 100) / 6) ** 2)
    z0 = O.als_baseline(y)[0]
    z1 = O.als_baseline(y + 5.0)[0]
    assert np.max(np.abs(z1 - z0 - 5.0)) < 1e-7
    zd = _als_dense(y, 1e4, 1e-3, 10)
    assert np.max(np.abs(z0 - zd)) < 1e-8


def test_P9b_als_hugs_baseline_below_positive_peaks():
    M = 800
    t = np.linspace(-1, 1, M)
    base = 0.2 + 0.3 * t - 0.25 * t * t
    peaks = sum(a / (1 + ((t - c) / 0.01) ** 2) for a, c in ((0.5, -0.5), (0.8, 0.1), (0.4, 0.6)))
    z = O.als_baseline(base + peaks)[0]
    away = np.ones(M, bool)
    for c in (-0.5, 0.1, 0.6):
        away &= np.abs(t - c) > 0.1
    assert np.sqrt(np.mean((z - base)[away] ** 2)) < 0.02 * np.ptp(base)


# ---------------------------------------------------------------- SG --------------------------
def test_P10_sg_quadratic_and_polyfit():
    M, w = 60, 21
    t = np.arange(M, dtype=float)
    q = 1.0 - 0.3 * t + 0.01 * t * t
    assert np.max(np.abs(O.sg_trend(q, w, 2)[0] - q)) < 1e-10
    rng = np.random.default_rng(5)
    y = rng.standard_normal(M)
    out = O.sg_trend(y, w, 2)[0]
    h = w // 2
    ref = np.empty(M)
    for i in range(M):
        lo = min(max(i - h, 0), M - w)
        c = np.polyfit(t[lo:lo + w], y[lo:lo + w], 2)
        ref[i] = np.polyval(c, t[i])
    assert np.max(np.abs(out - ref)) < 1e-10


def test_P16_sg_constant_rows():
    x = np.array([[1.5] * 100, [-2.0] * 100])
    assert np.max(np.abs(O.sg_trend(x, 75, 2) - x)) < 1e-12


# ---------------------------------------------------------------- SVD / factorized ------------
def test_P11_svd_full_rank_exact():
    rng = np.random.default_rng(6)
    A = rng.standard_normal((64, 32))
    V, s, _ = O.eig_topk(O.gram(A), 32)
    U, s_ref, Vt = np.linalg.svd(A, full_matrices=False)
    assert np.max(np.abs(s - s_ref)) / s_ref[0] < 1e-12
    assert np.max(np.abs(np.abs(V) - np.abs(Vt.T))) < 1e-10
    assert np.max(np.abs(V.T @ V - np.eye(32))) < 1e-12
    US = A @ V
    assert np.max(np.abs(US @ V.T - A)) < 1e-12          # U S V^T = A at full rank
    # sign rule: largest |entry| of each column positive
    assert np.all(V[np.argmax(np.abs(V), axis=0), np.arange(32)] > 0)


def test_rank_cutoff_golden():
    g = GOLD["rank_cutoff_example"]
    assert O.rank_cutoff(np.array(g["s"]), g["M"], g["N"], g["eps"]) == g["keep"]
    assert O.rank_cutoff(np.array([0.0]), 3, 3, 2.2e-16) == 0


def test_f_eq9_golden():
    for g in GOLD["f_eq9_examples"]:
        I = np.full((7, 5), g["mean_I"])
        p = O.Params(f_mode="eq9", f_alpha=g["alpha"], f_sigma_g=g["sigma_g"])
        assert np.allclose(O.noise_scale_f(I, p), g["f"], rtol=1e-14)
    assert np.all(O.noise_scale_f(np.ones((2, 3)), P0) == 1.0)


def test_log_ratio_rows():
    ref = np.array([1.0, 2.0, 0.5])
    A = O.log_ratio(np.vstack([ref, np.e ** 2 * ref]), ref, P0)
    assert np.max(np.abs(A[0])) < 1e-15 and np.max(np.abs(A[1] - 1.0)) < 1e-14


def _small_cube(N=200, M=64, seed=7):
    rng = np.random.default_rng(seed)
    w = np.linspace(0, 1, M)
    C = rng.uniform(0, 1, (N, 3))
    chi = sum(C[:, [s]] * (0.05 / (c - w[None, :] - 0.03j)) for s, c in enumerate((0.3, 0.5, 0.7)))
    I = np.abs(1 + chi) ** 2 * (1 + 0.01 * rng.standard_normal((N, M)))
    Iref = 1 + 0.2 * w
    return I, Iref


def test_P12_fkk_equals_kk_full_rank():
    """Eq. 7: H{A} = U S H{V^T}; at full rank, f == 1, no PEC/SEC,
    exp(A) exp(i US H{V^T}) equals the per-spectrum KK of Eq. 3."""
    I, Iref = _small_cube()
    A = O.log_ratio(I, Iref, P0)
    V, s, _ = O.eig_topk(O.gram(A), A.shape[1])
    US = A @ V
    K_f = np.exp(US @ V.T) * np.exp(1j * (US @ O.hilbert(V.T)))
    K_kk = O.kk(I, Iref, P0)
    assert np.max(np.abs(K_f - K_kk)) / np.max(np.abs(K_kk)) < 1e-10


def test_P13_gemm_route_equals_per_pixel_route():
    I, Iref = _small_cube(seed=8)
    k = 8
    out = O.fkk_ec(I, Iref, k, P0)
    US, V, f = out["US"], out["V"], out["f"]
    ak = US @ (V.T / f[None, :])
    phihat = US @ out["phi_pec"]
    amp = ak + O.hilbert(phihat)
    amp = amp - O.sg_trend(amp, O.sg_window(I.shape[1], P0), 2)
    ph = O.hilbert(ak) - phihat
    K_pix = np.exp(amp) * np.exp(1j * ph)
    assert np.max(np.abs(K_pix - out["K"])) / np.max(np.abs(out["K"])) < 1e-10


def test_P14_ml_closed_form_and_self_consistency():
    I, Iref = _small_cube(seed=9)
    k = 10
    for rel in (1e-2, 1e-6):
        p = O.Params(ml_ridge_rel=rel)
        out = O.fkk_ec(I, Iref, k, p)
        W = O.ml_projector(out["V"], out["s"], p)
        Wg = O.ml_projector_general(out["V"], out["s"], p)
        assert np.max(np.abs(W - Wg)) / np.max(np.abs(W)) < 1e-8
    model, K_train = O.ml_train(I, Iref, k, P0)
    K_apply = O.ml_apply(I, Iref, model, P0)
    assert np.max(np.abs(K_apply - K_train)) / np.max(np.abs(K_train)) < 1e-10


def test_P15_fpec_trivia():
    rng = np.random.default_rng(10)
    X = rng.standard_normal((12, 5))
    assert np.max(np.abs(O.ridge_solve(X, np.zeros((12, 30)), 0.1))) == 0.0
    Y = rng.standard_normal((5, 30))
    assert np.max(np.abs(O.ridge_solve(np.eye(5), Y, 0.0) - Y)) < 1e-14
    # general ridge equals the normal-equation least squares at lam=0
    Y2 = rng.standard_normal((12, 30))
    ls = np.linalg.lstsq(X, Y2, rcond=None)[0]
    assert np.max(np.abs(O.ridge_solve(X, Y2, 0.0) - ls)) < 1e-9


def test_P18_sign_freedom():
    I, Iref = _small_cube(seed=11)
    k = 6
    out = O.fkk_ec(I, Iref, k, P0)
    flip = np.array([1, -1, 1, -1, -1, 1.0])
    out2 = O.fkk_ec_from(I, Iref, out["V"] * flip[None, :], out["s"], out["q"], P0)
    assert np.max(np.abs(out2["K"] - out["K"])) / np.max(np.abs(out["K"])) < 1e-12


def test_select_q_union_and_ties():
    US = np.array([[1.0, -2.0], [3.0, 5.0], [3.0, -2.0], [-1.0, 0.0]])
    # col0: max 3 at rows 1,2 -> 1 ; min -1 at 3.  col1: max 5 at 1 ; min -2 at rows 0,2 -> 0
    assert list(O.select_q(US)) == [0, 1, 3]


# ---------------------------------------------------------------- sizes / quality -------------
def test_P19_paper_sizes():
    g = GOLD["sim_base_pixels"]["value"]
    assert g[0] * g[1] == g[2]
    base_h, base_w = g[0], g[1]
    for sc, tot in zip(GOLD["sim_side_scaled_totals"]["scales"], GOLD["sim_side_scaled_totals"]["value"]):
        assert int(round(base_h * sc)) * int(round(base_w * sc)) == tot
    t = GOLD["tissue_pixels"]["value"]
    assert t[0] * t[1] == t[2] == CONFIGS["cfg3"].n_pixels


def test_P20_quality_cfg1():
    """fKK-EC <RSS> well below Null RSS on the tiny config (Fig. 2e claim)."""
    cfg = CONFIGS["cfg1"]
    I, Iref, _ = generate(cfg)
    out = O.fkk_ec(I, Iref, cfg.rank_k, P0)
    truth = truth_imag(cfg)
    r = O.rss(out["K"], truth).mean()
    null = O.rss(np.zeros_like(out["K"]), truth).mean()
    assert r < 0.1 * null


# ------------------------------------------------------------------ conventional workflow (NEXT row 2)
def test_P21_svd_denoise_eckart_young_and_full_rank():
    """svd_denoise against the SVD definition: the truncation error is the tail of the singular values
    (Eckart-Young, ||I - I_k||_F^2 = sum_{i>k} sigma_i^2 from numpy.linalg.svd), I_k has rank k, full
    rank reproduces I, and a rank-1 cube is reproduced at k = 1."""
    rng = np.random.default_rng(5)
    I = rng.random((40, 24)) + 0.5
    sig = np.linalg.svd(I, compute_uv=False)
    for k in (1, 3, 7):
        Ik = O.svd_denoise(I, k)
        assert abs(np.sum((I - Ik) ** 2) - np.sum(sig[k:] ** 2)) <= 1e-9 * np.sum(sig ** 2)
        assert np.linalg.matrix_rank(Ik, tol=1e-9 * sig[0]) == k
    assert np.max(np.abs(O.svd_denoise(I, 24) - I)) <= 1e-12 * np.max(np.abs(I))
    r1 = np.outer(rng.random(30) + 0.5, rng.random(24) + 0.5)
    assert np.max(np.abs(O.svd_denoise(r1, 1) - r1)) <= 1e-12 * np.max(r1)


def test_P22_conventional_full_rank_equals_direct():
    """At full rank the SVD denoise is the identity, so the conventional workflow equals kk_direct."""
    from synth import CONFIGS, generate
    cfg = CONFIGS["cfg1"].with_(height=3, width=4, n_freq=64)
    I, Iref, _ = generate(cfg)
    K_conv = O.conventional_workflow(I, Iref, 64)
    K_dir = O.kk_direct(I, Iref)
    assert np.max(np.abs(K_conv - K_dir)) <= 1e-9 * np.max(np.abs(K_dir))
