"""fp64 CPU oracle for fKK-EC (arxiv 2005.07132) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this module.  The product path (``paper_2005_07132_b200``) never does,
and this module never imports the product path: the two share no code.

Every function is the plain, slow, obviously-correct statement of one step, in the paper's order
and notation, in float64 (NumPy; SciPy's banded Cholesky as the one library primitive for ALS).
Citations are ``PAPER.md:<line> (section, Eq.)``; readings where the paper is silent are the
DESIGN.md "Readings" table (A1..A24).  Letters follow BASELINE.json: N spectra (rows) x M channels.

Parity status: every public function here is pinned by tests/test_oracle_pins.py except where its
docstring says "parity unpinned".
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.linalg

# ----------------------------------------------------------------------------------------------
# Parameters (readings A3, A6, A8, A11, A16)
# ----------------------------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class Params:
    pad: str = "reflect"          # A3: "reflect" (default) | "zero" | "none" (L == M, periodic)
    fft_len: int = 0              # 0 -> L = 2 * nextpow2(M)
    ratio_floor: float = 1e-6     # A16: clamp of I/I_ref before ln
    als_lambda: float = 1e4       # A6
    als_p: float = 1e-3           # A6
    als_iters: int = 10           # A6
    sg_window: int = 0            # A8: 0 -> 2*floor(0.375*M)+1
    sg_order: int = 2             # A8
    ridge_rel: float = 1e-3       # A11: lambda = ridge_rel * lambda_max(X^T X)
    ml_ridge_rel: float = 0.0     # Eq. 25 ridge, lambda_ml = ml_ridge_rel * s_1^2
    f_mode: str = "one"           # A15: "one" | "eq9"
    f_alpha: float = 0.0
    f_sigma_g: float = 1.0


def fft_length(M: int, p: Params) -> int:
    if p.pad == "none":
        return M
    if p.fft_len:
        return p.fft_len
    return 2 * (1 << int(np.ceil(np.log2(M))))


def sg_window(M: int, p: Params) -> int:
    return p.sg_window if p.sg_window else 2 * int(np.floor(0.375 * M)) + 1


# ----------------------------------------------------------------------------------------------
# F0 / F1: noise scaling and log-ratio matrix
# ----------------------------------------------------------------------------------------------


def noise_scale_f(I: np.ndarray, p: Params) -> np.ndarray:
    """f(omega), PAPER.md:97-99 (Eq. 9): f = 2<I> / sqrt(alpha <I> + sigma_g^2); f == 1 when
    p.f_mode == "one" ("can be set to one")."""
    M = I.shape[1]
    if p.f_mode == "one":
        return np.ones(M)
    mean = np.asarray(I, dtype=np.float64).mean(axis=0)
    return 2.0 * mean / np.sqrt(p.f_alpha * mean + p.f_sigma_g ** 2)


def log_ratio(I: np.ndarray, I_ref: np.ndarray, p: Params, f: np.ndarray | None = None) -> np.ndarray:
    """A[n, j] = f_j * 1/2 * ln(I[n, j] / I_ref[j])  -- PAPER.md:66-68 (Eq. 6), :103 (Eq. 10).
    The ratio is clamped below at p.ratio_floor (reading A16)."""
    r = np.asarray(I, dtype=np.float64) / np.asarray(I_ref, dtype=np.float64)[None, :]
    a = 0.5 * np.log(np.maximum(r, p.ratio_floor))
    if f is not None:
        a = a * f[None, :]
    return a


# ----------------------------------------------------------------------------------------------
# Hilbert transform ("Hilbert transform"; padding reading A3; sign reading A2)
# ----------------------------------------------------------------------------------------------


def hilbert(x: np.ndarray, p: Params = Params()) -> np.ndarray:
    """Row-wise discrete Hilbert transform H{x} with H{cos} = sin, H{sin} = -cos (A2).

    Each length-M row is extended to L samples (centred: pl = floor((L-M)/2) on the left),
    by even reflection without repeating the edge sample (REFLECT, numpy 'reflect') or by zeros
    (ZERO); "none" requires L == M (periodic).  X = DFT_L(x_ext); multiply by h with h[0] = h[L/2]
    = 0 (A4), h[j] = -i for 0 < j < L/2, +i for L/2 < j < L; H{x} = Re(IDFT_L(h X))[pl:pl+M].
    """
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    M = x.shape[1]
    L = fft_length(M, p)
    pl = (L - M) // 2
    pr = L - M - pl
    if p.pad == "reflect":
        xe = np.pad(x, ((0, 0), (pl, pr)), mode="reflect")
    elif p.pad == "zero":
        xe = np.pad(x, ((0, 0), (pl, pr)), mode="constant")
    elif p.pad == "none":
        assert L == M
        xe = x
    else:
        raise ValueError(p.pad)
    X = np.fft.fft(xe, axis=1)
    h = np.zeros(L, dtype=np.complex128)
    h[1:L // 2] = -1j
    h[L // 2 + 1:] = 1j
    out = np.fft.ifft(X * h[None, :], axis=1).real
    return out[:, pl:pl + M]


# ----------------------------------------------------------------------------------------------
# ALS detrending D{.} ("asymmetric least squares (ALS)"; reading A6, A7)
# ----------------------------------------------------------------------------------------------


def als_matrix_bands(M: int, lam: float, w: np.ndarray) -> np.ndarray:
    """Upper banded form (3 x M) of W + lam D^T D, D the (M-2) x M second-difference operator."""
    D = np.zeros((M - 2, M))
    for i in range(M - 2):
        D[i, i], D[i, i + 1], D[i, i + 2] = 1.0, -2.0, 1.0
    DtD = D.T @ D
    ab = np.zeros((3, M))
    ab[2] = np.diag(DtD) * lam + w
    ab[1, 1:] = np.diag(DtD, 1) * lam
    ab[0, 2:] = np.diag(DtD, 2) * lam
    return ab


def als_baseline(y: np.ndarray, p: Params = Params()) -> np.ndarray:
    """Asymmetric least squares baseline (Eilers' Whittaker smoother with asymmetric weights):
    minimise sum_i w_i (y_i - z_i)^2 + lam sum_i (z_{i-1} - 2 z_i + z_{i+1})^2, i.e. solve
    (W + lam D^T D) z = W y; w^0 = 1; after each solve w_i = p if y_i > z_i else 1 - p.
    Exactly p.als_iters solves, all fp64 (A6, A7).  Rows of a 2-D input are independent."""
    y2 = np.atleast_2d(np.asarray(y, dtype=np.float64))
    N, M = y2.shape
    out = np.empty_like(y2)
    for n in range(N):
        yn = y2[n]
        w = np.ones(M)
        z = yn
        for _ in range(p.als_iters):
            ab = als_matrix_bands(M, p.als_lambda, w)
            z = scipy.linalg.solveh_banded(ab, w * yn)
            w = np.where(yn > z, p.als_p, 1.0 - p.als_p)
        out[n] = z
    return out


# ----------------------------------------------------------------------------------------------
# Trendline M{.}: large-window, low-order Savitzky-Golay (reading A8)
# ----------------------------------------------------------------------------------------------


def sg_trend(y: np.ndarray, window: int, order: int = 2) -> np.ndarray:
    """Savitzky-Golay trend of each row: interior point i -> value at i of the least-squares
    polynomial (degree `order`) through y[i-h .. i+h]; the first/last h points -> the polynomial
    fitted to the first/last `window` samples evaluated there ("polynomial edge handling")."""
    y2 = np.atleast_2d(np.asarray(y, dtype=np.float64))
    N, M = y2.shape
    w = min(window, M if M % 2 else M - 1)
    h = (w - 1) // 2
    k = np.arange(-h, h + 1, dtype=np.float64)
    V = np.vander(k, order + 1, increasing=True)          # w x (order+1)
    Vp = np.linalg.pinv(V)                                 # (order+1) x w
    centre = Vp[0]                                         # value at k=0
    out = np.empty_like(y2)
    idx = np.arange(h, M - h)
    win = idx[:, None] + np.arange(-h, h + 1)[None, :]
    for n in range(N):
        out[n, h:M - h] = y2[n, win] @ centre
    # edges: fit on first / last w samples, evaluate at the first / last h points
    ke = np.arange(w, dtype=np.float64) - h
    Ve = np.vander(ke, order + 1, increasing=True)
    coef_lo = Vp @ y2[:, :w].T                             # (order+1) x N
    coef_hi = Vp @ y2[:, M - w:].T
    out[:, :h] = (Ve[:h] @ coef_lo).T
    out[:, M - h:] = (Ve[w - h:] @ coef_hi).T
    return out


# ----------------------------------------------------------------------------------------------
# Direct (conventional) path, per spectrum: D1..D5 (Eqs. 2-5)
# ----------------------------------------------------------------------------------------------


def kk(I: np.ndarray, I_ref: np.ndarray, p: Params = Params()) -> np.ndarray:
    """K = sqrt(I/I_ref) exp(i H{1/2 ln(I/I_ref)})  -- PAPER.md:42 (Eq. 3)."""
    a = log_ratio(I, I_ref, p)
    phi = hilbert(a, p)
    return np.exp(a + 1j * phi)


def kk_direct(I: np.ndarray, I_ref: np.ndarray, p: Params = Params(), stages: dict | None = None
              ) -> np.ndarray:
    """Conventional KK + PEC + SEC, PAPER.md:53 (Eq. 5) in the log domain:
       a = 1/2 ln(I/I_ref);  phi = H{a};  phi_err = D{phi} (ALS);
       a' = a + H{phi_err};  phi' = phi - phi_err;  K' = exp(a') (cos phi' + i sin phi');
       T = M{Re K'} (SG trend; the scalar mean if min T <= 0, reading A9);  K_CARS = K' / T."""
    a = log_ratio(I, I_ref, p)
    phi = hilbert(a, p)
    phi_err = als_baseline(phi, p)
    a2 = a + hilbert(phi_err, p)
    phi2 = phi - phi_err
    K1 = np.exp(a2) * (np.cos(phi2) + 1j * np.sin(phi2))
    T = sg_trend(K1.real, sg_window(a.shape[1], p), p.sg_order)
    bad = T.min(axis=1) <= 0
    if np.any(bad):
        T[bad] = K1.real[bad].mean(axis=1, keepdims=True)
    if stages is not None:
        stages.update(a=a, phi=phi, phi_err=phi_err, T=T)
    return K1 / T


# ----------------------------------------------------------------------------------------------
# Factorized path F0..F11 and ML reuse F12
# ----------------------------------------------------------------------------------------------


def gram(A: np.ndarray) -> np.ndarray:
    """G = A^T A (M x M, uncentred; reading A17) -- the normal matrix of the SVD A = U S V^T."""
    return A.T @ A


def eig_topk(G: np.ndarray, k: int):
    """Truncated SVD through the Gram matrix: G = V Lambda V^T, keep the k
    largest eigenpairs; s = sqrt(lambda).  Sign rule: in each column the entry of largest |.| is
    made positive (ties -> lowest index).  Returns (V_k [M x k], s [k], all eigenvalues desc)."""
    lam, V = np.linalg.eigh(G)
    order = np.argsort(lam)[::-1]
    lam = lam[order]
    V = V[:, order[:k]].copy()
    for i in range(k):
        j = int(np.argmax(np.abs(V[:, i])))
        if V[j, i] < 0:
            V[:, i] = -V[:, i]
    return V, np.sqrt(np.maximum(lam[:k], 0.0)), lam


def rank_cutoff(s: np.ndarray, M: int, N: int, eps: float) -> int:
    """Count of s_i > s_max * max(M, N) * eps (reading A14: "max A" = sigma_max,
    the NumPy/MATLAB matrix_rank rule)."""
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        return 0
    return int(np.sum(s > s.max() * max(M, N) * eps))


def select_q(US: np.ndarray) -> np.ndarray:
    """q = q_max U q_min: per column argmax / argmin of U (equivalently of US since s > 0),
    PAPER.md:117-121 (Eqs. 13-15); ties -> lowest row; sorted ascending, unique (A12)."""
    qmax = np.argmax(US, axis=0)
    qmin = np.argmin(US, axis=0)
    return np.unique(np.concatenate([qmax, qmin]))


def lambda_max_sym(C: np.ndarray) -> float:
    return float(np.linalg.eigvalsh(C)[-1])


def fpec(X: np.ndarray, Hv: np.ndarray, p: Params):
    """fPEC, PAPER.md:123-125 (Eqs. 16-17): Phi_err = D{X H{V^T/f}} (ALS on each row),
    Phi_PEC^T = (X^T X + lambda I)^{-1} X^T Phi_err, lambda = ridge_rel * lambda_max(X^T X) (A11).
    Returns (Phi_err, Phi_PEC^T, lambda)."""
    P = X @ Hv
    phi_err = als_baseline(P, p)
    C = X.T @ X
    lam = p.ridge_rel * lambda_max_sym(C)
    phi_pec = ridge_solve(X, phi_err, lam)
    return phi_err, phi_pec, lam


def ridge_solve(X: np.ndarray, Y: np.ndarray, lam: float) -> np.ndarray:
    """(X^T X + lam I)^{-1} X^T Y via Cholesky (Eq. 17)."""
    C = X.T @ X + lam * np.eye(X.shape[1])
    c = scipy.linalg.cho_factor(C)
    return scipy.linalg.cho_solve(c, X.T @ Y)


def basis(V: np.ndarray, s: np.ndarray, f: np.ndarray, X: np.ndarray, p: Params) -> dict:
    """F6..F10 on the k basis vectors:
       Hv = H{V^T/f}                                      (Eq. 11)
       Phi_err, Phi_PEC^T                                 (Eqs. 16-17)
       HPhi = H{Phi_PEC^T}                                (Eq. 18)
       V_SEC^T = M{V^T/f + HPhi}   (row-wise SG trend)    (Eq. 22)
       B_amp = V^T/f + HPhi - V_SEC^T;  B_ph = Hv - Phi_PEC^T     (Eq. 23)."""
    Vt_f = V.T / f[None, :]
    Hv = hilbert(Vt_f, p)
    phi_err, phi_pec, lam = fpec(X, Hv, p)
    HPhi = hilbert(phi_pec, p)
    v_sec = sg_trend(Vt_f + HPhi, sg_window(V.shape[0], p), p.sg_order)
    B_amp = Vt_f + HPhi - v_sec
    B_ph = Hv - phi_pec
    return dict(Hv=Hv, phi_err=phi_err, phi_pec=phi_pec, ridge_lambda=lam, HPhi=HPhi,
                v_sec=v_sec, B_amp=B_amp, B_ph=B_ph)


def reconstruct(US: np.ndarray, B_amp: np.ndarray, B_ph: np.ndarray) -> np.ndarray:
    """K_CARS = exp[US B_amp] exp[i US B_ph]  -- PAPER.md:162 (Eq. 23)."""
    return np.exp(US @ B_amp) * np.exp(1j * (US @ B_ph))


def fkk_ec(I: np.ndarray, I_ref: np.ndarray, k: int, p: Params = Params()) -> dict:
    """Full fKK-EC, Fig. 1(b): F0..F11.  Returns every stage (for stage-wise parity)."""
    f = noise_scale_f(I, p)
    A = log_ratio(I, I_ref, p, f)
    G = gram(A)
    V, s, lam_all = eig_topk(G, k)
    US = A @ V
    q = select_q(US)
    out = fkk_ec_from(I, I_ref, V, s, q, p, f=f, A=A)
    out.update(f=f, G=G, V=V, s=s, eigvals=lam_all)
    return out


# ----------------------------------------------------------------------------------------------
# Randomized range finder SVD ("random sampling ('randomized') SVD
# ... [Halko 2011]"): randomized subspace iteration followed by the SVD of the small projected matrix.
# ----------------------------------------------------------------------------------------------


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 counters (Steele, Lea & Flood 2014): the counter-based generator
    the range finder draws its test matrix from (the CUDA library implements the same function)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def range_finder_omega(seed: int, M: int, l: int) -> np.ndarray:
    """Gaussian test matrix Omega (M x l) by Box-Muller from two SplitMix64 draws per entry:
    u1 = (h(2c) >> 11 + 1) / 2^53, u2 = (h(2c+1) >> 11) / 2^53 with counter c = seed * 2^40 + j * l + i
    for entry (j, i);  Omega[j, i] = sqrt(-2 ln u1) cos(2 pi u2)."""
    j, i = np.meshgrid(np.arange(M, dtype=np.uint64), np.arange(l, dtype=np.uint64), indexing="ij")
    c = np.uint64(seed) * np.uint64(1 << 40) + j * np.uint64(l) + i
    h1 = splitmix64(np.uint64(2) * c)
    h2 = splitmix64(np.uint64(2) * c + np.uint64(1))
    u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) / 9007199254740992.0
    u2 = (h2 >> np.uint64(11)).astype(np.float64) / 9007199254740992.0
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def _orth(Y: np.ndarray) -> np.ndarray:
    """Orthonormal basis of range(Y) (Householder QR, numpy.linalg.qr)."""
    return np.linalg.qr(Y)[0]


def randomized_svd(A: np.ndarray, k: int, omega: np.ndarray, q: int) -> tuple[np.ndarray, np.ndarray]:
    """Halko, Martinsson & Tropp (2011), Alg. 4.4 (randomized subspace iteration) + Alg. 5.1 (direct
    SVD): Y = A Omega; Q = orth(Y); q times {Q = orth(A orth(A^T Q))}; B = Q^T A; B = U~ S V^T.
    Returns V_k (M x k, the sign rule of eig_topk) and s_k."""
    Q = _orth(A @ omega)
    for _ in range(q):
        Q = _orth(A.T @ Q)
        Q = _orth(A @ Q)
    B = Q.T @ A
    _, sv, Vt = np.linalg.svd(B, full_matrices=False)
    V = Vt[:k].T.copy()
    for i in range(k):
        jmax = int(np.argmax(np.abs(V[:, i])))
        if V[jmax, i] < 0:
            V[:, i] = -V[:, i]
    return V, sv[:k]


def fkk_ec_randomized(I: np.ndarray, I_ref: np.ndarray, k: int, oversample: int, q: int, seed: int,
                      p: Params = Params()) -> dict:
    """fKK-EC with the randomized range finder in place of the Gram eigensolver (F2-F4), then F5..F11
    as fkk_ec (PAPER.md:226 with Fig. 1(b))."""
    f = noise_scale_f(I, p)
    A = log_ratio(I, I_ref, p, f)
    omega = range_finder_omega(seed, A.shape[1], k + oversample)
    V, s = randomized_svd(A, k, omega, q)
    US = A @ V
    qq = select_q(US)
    out = fkk_ec_from(I, I_ref, V, s, qq, p, f=f, A=A)
    out.update(f=f, V=V, s=s, omega=omega)
    return out


def fkk_ec_from(I, I_ref, V, s, q, p: Params = Params(), f=None, A=None) -> dict:
    """F5..F11 with a given V_k, s and q (stage-wise parity, DESIGN.md parity contract)."""
    if f is None:
        f = noise_scale_f(I, p)
    if A is None:
        A = log_ratio(I, I_ref, p, f)
    US = A @ V
    X = US[np.asarray(q)]
    b = basis(V, s, f, X, p)
    K = reconstruct(US, b["B_amp"], b["B_ph"])
    b.update(US=US, q=np.asarray(q), X=X, K=K, f=f)
    return b


def ml_projector(V: np.ndarray, s: np.ndarray, p: Params) -> np.ndarray:
    """Eq. 25 in closed form: with X = S V^T and V^T V = I,
    (X^T X + lam I)^{-1} X^T ... applied as U_new S = A_new W, W = V diag(s^2/(s^2+lam)),
    lam = ml_ridge_rel * s_1^2."""
    lam = p.ml_ridge_rel * s[0] ** 2
    return V * (s ** 2 / (s ** 2 + lam))[None, :]


def ml_projector_general(V: np.ndarray, s: np.ndarray, p: Params) -> np.ndarray:
    """Eq. 25 literally: U_new = A_new (X^T X + lam I)^{-1} X^T with X = S V^T
    (k x M), an M x M ridge system (lam > 0; for lam = 0 the minimum-norm least-squares solution
    A_new pinv(X)).  Returns the M x k matrix W_g with U_new S = A_new W_g (comparable to W)."""
    X = np.diag(s) @ V.T
    lam = p.ml_ridge_rel * s[0] ** 2
    M = X.shape[1]
    if lam > 0:
        Wt = np.linalg.solve(X.T @ X + lam * np.eye(M), X.T)   # M x k
    else:
        Wt = np.linalg.pinv(X)                                  # M x k
    return Wt * s[None, :]


def ml_apply(I_new: np.ndarray, I_ref: np.ndarray, model: dict, p: Params = Params()) -> np.ndarray:
    """ML:fKK-EC: A_new = f/2 ln(I_new/I_ref); US_new = A_new W; then Eq. 23 with
    the trained B_amp, B_ph."""
    A = log_ratio(I_new, I_ref, p, model["f"])
    US = A @ model["W"]
    return reconstruct(US, model["B_amp"], model["B_ph"])


def ml_train(I, I_ref, k, p: Params = Params()) -> tuple[dict, np.ndarray]:
    out = fkk_ec(I, I_ref, k, p)
    model = dict(f=out["f"], V=out["V"], s=out["s"], W=ml_projector(out["V"], out["s"], p),
                 B_amp=out["B_amp"], B_ph=out["B_ph"], I_ref=np.asarray(I_ref, np.float64))
    return model, out["K"]


# ----------------------------------------------------------------------------------------------
# Quality metric (harness): RSS against known Im{chi/chi_nr}
# ----------------------------------------------------------------------------------------------


def svd_denoise(I: np.ndarray, k: int) -> np.ndarray:
    """Rank-k SVD denoise of the RAW cube (the conventional workflow's first step, Fig. 1(a),
    PAPER.md:58, :64 "creating new U, S and V matrices that exclude the non-desired singular values";
    the conventional SVD acts on raw BCARS spectra, not on the log-ratio):
    I_k = U_k S_k V_k^T = (I V_k) V_k^T with V_k the top-k eigenvectors of I^T I (reading A26)."""
    V, _, _ = eig_topk(gram(I), k)
    return (I @ V) @ V.T


def conventional_workflow(I: np.ndarray, I_ref: np.ndarray, k: int, p: Params = Params()) -> np.ndarray:
    """The paper's comparison baseline (Fig. 1(a)): SVD denoise of the raw
    cube to rank k, then the per-spectrum KK + PEC + SEC (kk_direct) of every denoised spectrum."""
    return kk_direct(svd_denoise(I, k), I_ref, p)


def rss(K: np.ndarray, truth_im: np.ndarray) -> np.ndarray:
    """Per-pixel sum over omega of (Im K - truth)^2.  Null RSS = rss(0, truth)."""
    return np.sum((np.imag(K) - truth_im) ** 2, axis=1)
