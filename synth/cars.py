"""Seeded synthetic CARS cubes (input generator shared by the oracle tests and the CUDA path).

This module holds the *physics of the measurement* only -- the CARS intensity model of
PAPER.md:32 (Eq. 1, right-hand side), the surrogate-reference error model of PAPER.md:40
(I_ref = Xi * xi(omega) * I_NRB) and additive Gaussian noise.  It contains none of the method's
arithmetic (no log-ratio, Hilbert transform, SVD, ALS, Savitzky-Golay, ridge): those live in
``oracle/`` (fp64 reference) and in the CUDA library, which never import each other.

Readings (SURVEY.md 8(d) marks them (R)):
  * axis omega_j = linspace(500, 3800, M) cm^-1, ascending; x_j = 2(omega_j-500)/3300 - 1.
  * species s: chi_R,s = r_s Gamma_s / (Omega_s - omega - i Gamma_s), Omega_s ~ U(500,3800),
    Gamma_s ~ U(5,20) (HWHM), r_s ~ U(0.2,1.0)  (so Im{chi_R,s} peaks at r_s; PAPER.md:140 form).
  * concentration fields: sum of 3 isotropic 2-D Gaussians (centres U(0,1)^2, widths
    U(0.08,0.3)*max(H,W)), normalised to max 1.  "mixed" configs combine n_fields fields into the
    species through B ~ U(0,1)^{fields x species}; otherwise one field per species.
  * NRB chi_NR = 1 (real constant) or exp(i theta(omega)) with theta = 0.1 rad * (Legendre series of
    degree <= 2, coefficients U(-1,1), normalised to max |.| = 1): the "slowly varying phase offset".
  * excitation profile P(omega) = exp(-(x-x0)^2/(2 sigma^2)) (1 + a1 x + a2 x^2) (C_st of Eq. 1).
  * clean intensity I0 = |chi_R + chi_NR|^2 P;  noise sigma_j = |chi_NR|^2 P_j / SNR (the NRB level
    per channel), I = I0 + sigma_j N(0,1).
  * reference I_ref = |chi_NR|^2 P xi,  xi = 1 + e tanh(sum_{d<=3} c_d P_d(x)), c_d ~ U(-1,1).
  * RNG: numpy Philox keyed by (seed, stream, 65,536-row block) so the cube does not depend on how
    it is chunked; "instrument" draws (species, P, xi, theta) use species_seed.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

BLOCK_ROWS = 65536
_STREAM_INSTRUMENT = 1
_STREAM_FIELDS = 2
_STREAM_MIX = 3
_STREAM_NOISE = 4


@dataclasses.dataclass(frozen=True)
class CubeConfig:
    name: str
    height: int
    width: int
    n_freq: int
    n_species: int
    n_fields: int
    mixed: bool            # fields mixed into species through B ~ U(0,1)
    snr: float
    xi_err: float          # e: surrogate-reference error amplitude
    phase_offset: bool     # chi_NR = exp(i theta(omega))
    seed: int
    species_seed: int
    rank_k: int
    dtype: str             # "f32" or "f64"
    omega_lo: float = 500.0
    omega_hi: float = 3800.0

    @property
    def n_pixels(self) -> int:
        return self.height * self.width

    def with_(self, **kw) -> "CubeConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; SURVEY.md 8(d) table.
CONFIGS = {
    "cfg1": CubeConfig("cfg1", 64, 64, 512, 6, 3, True, 50.0, 0.10, False, 0, 0, 12, "f64"),
    "cfg2": CubeConfig("cfg2", 256, 256, 1000, 10, 4, True, 20.0, 0.20, False, 0, 0, 40, "f32"),
    "cfg3": CubeConfig("cfg3", 846, 831, 1000, 12, 12, False, 10.0, 0.20, True, 0, 0, 60, "f32"),
    "cfg4": CubeConfig("cfg4", 2000, 2000, 1600, 16, 16, False, 10.0, 0.20, False, 0, 0, 100, "f32"),
    # config 5: training cube = config-2 generator with seed 1 / species_seed 1; apply cube = a
    # 703,026-pixel cube of the same instrument (species, P, xi) with new fields and noise (seed 2).
    "cfg5_train": CubeConfig("cfg5_train", 256, 256, 1000, 10, 4, True, 20.0, 0.20, False, 1, 1, 40, "f32"),
    "cfg5_apply": CubeConfig("cfg5_apply", 846, 831, 1000, 10, 4, True, 20.0, 0.20, False, 2, 1, 40, "f32"),
}


def _rng(seed: int, stream: int, block: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed), (int(stream) << 40) | int(block)]))


def omega_axis(cfg: CubeConfig) -> np.ndarray:
    return np.linspace(cfg.omega_lo, cfg.omega_hi, cfg.n_freq)


def _xnorm(cfg: CubeConfig) -> np.ndarray:
    w = omega_axis(cfg)
    return 2.0 * (w - cfg.omega_lo) / (cfg.omega_hi - cfg.omega_lo) - 1.0


def _legendre(x: np.ndarray, deg: int) -> list[np.ndarray]:
    out = [np.ones_like(x), x.copy()]
    for n in range(1, deg):
        out.append(((2 * n + 1) * x * out[n] - n * out[n - 1]) / (n + 1))
    return out[: deg + 1]


@dataclasses.dataclass
class Instrument:
    omega: np.ndarray        # M
    chi_species: np.ndarray  # S x M complex128
    chi_nr: np.ndarray       # M complex128
    profile: np.ndarray      # M, P(omega) > 0
    xi: np.ndarray           # M, surrogate error xi(omega) > 0
    centres: np.ndarray
    widths: np.ndarray
    ratios: np.ndarray


def instrument(cfg: CubeConfig) -> Instrument:
    g = _rng(cfg.species_seed, _STREAM_INSTRUMENT)
    w = omega_axis(cfg)
    x = _xnorm(cfg)
    S = cfg.n_species
    centres = g.uniform(cfg.omega_lo, cfg.omega_hi, S)
    widths = g.uniform(5.0, 20.0, S)
    ratios = g.uniform(0.2, 1.0, S)
    chi = (ratios * widths)[:, None] / (centres[:, None] - w[None, :] - 1j * widths[:, None])
    x0, sig = g.uniform(-0.2, 0.2), g.uniform(0.8, 1.2)
    a1, a2 = g.uniform(-0.3, 0.3), g.uniform(-0.2, 0.2)
    profile = np.exp(-((x - x0) ** 2) / (2 * sig * sig)) * (1.0 + a1 * x + a2 * x * x)
    c = g.uniform(-1.0, 1.0, 4)
    leg = _legendre(x, 3)
    xi = 1.0 + cfg.xi_err * np.tanh(sum(c[d] * leg[d] for d in range(4)))
    th = g.uniform(-1.0, 1.0, 3)
    if cfg.phase_offset:
        theta = sum(th[d] * leg[d] for d in range(3))
        theta = 0.1 * theta / np.max(np.abs(theta))
        chi_nr = np.exp(1j * theta)
    else:
        chi_nr = np.ones(cfg.n_freq, dtype=np.complex128)
    return Instrument(w, chi, chi_nr, profile, xi, centres, widths, ratios)


def _fields_grid(cfg: CubeConfig) -> np.ndarray:
    """n_fields x (H*W) concentration fields, each normalised to max 1."""
    g = _rng(cfg.seed, _STREAM_FIELDS)
    H, W = cfg.height, cfg.width
    yy = np.arange(H, dtype=np.float64)[:, None]
    xx = np.arange(W, dtype=np.float64)[None, :]
    L = float(max(H, W))
    out = np.empty((cfg.n_fields, H * W))
    for f in range(cfg.n_fields):
        fld = np.zeros((H, W))
        for _ in range(3):
            cy, cx = g.uniform(0, 1) * H, g.uniform(0, 1) * W
            s = g.uniform(0.08, 0.3) * L
            fld += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
        out[f] = (fld / fld.max()).ravel()
    return out


def concentrations(cfg: CubeConfig) -> np.ndarray:
    """(H*W) x S species concentrations."""
    fl = _fields_grid(cfg)
    if cfg.mixed:
        B = _rng(cfg.seed, _STREAM_MIX).uniform(0.0, 1.0, (cfg.n_fields, cfg.n_species))
        return fl.T @ B
    assert cfg.n_fields == cfg.n_species
    return np.ascontiguousarray(fl.T)


def reference(cfg: CubeConfig, inst: Instrument | None = None) -> np.ndarray:
    """Surrogate reference I_ref = |chi_NR|^2 P xi, length M, fp64."""
    inst = inst or instrument(cfg)
    return np.abs(inst.chi_nr) ** 2 * inst.profile * inst.xi


def _block(cfg, inst, conc, b, out, dtype):
    r0 = b * BLOCK_ROWS
    r1 = min(cfg.n_pixels, r0 + BLOCK_ROWS)
    c = conc[r0:r1]
    re = c @ inst.chi_species.real + inst.chi_nr.real[None, :]
    im = c @ inst.chi_species.imag + inst.chi_nr.imag[None, :]
    i0 = (re * re + im * im) * inst.profile[None, :]
    sigma = np.abs(inst.chi_nr) ** 2 * inst.profile / cfg.snr
    noise = _rng(cfg.seed, _STREAM_NOISE, b).standard_normal((r1 - r0, cfg.n_freq))
    i0 += noise * sigma[None, :]
    out[r0:r1] = i0.astype(dtype, copy=False)


def generate(cfg: CubeConfig, threads: int | None = None):
    """Return (I [N x M] in cfg.dtype, I_ref [M] in cfg.dtype, omega [M] fp64)."""
    inst = instrument(cfg)
    conc = concentrations(cfg)
    dtype = np.float64 if cfg.dtype == "f64" else np.float32
    out = np.empty((cfg.n_pixels, cfg.n_freq), dtype=dtype)
    nb = (cfg.n_pixels + BLOCK_ROWS - 1) // BLOCK_ROWS
    threads = threads or min(nb, max(1, len(os.sched_getaffinity(0))))
    if threads <= 1 or nb == 1:
        for b in range(nb):
            _block(cfg, inst, conc, b, out, dtype)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda b: _block(cfg, inst, conc, b, out, dtype), range(nb)))
    return out, reference(cfg, inst).astype(dtype), inst.omega


def generate_rows(cfg: CubeConfig, r0: int, r1: int, threads: int | None = None):
    """Rows [r0, r1) of generate(cfg)'s cube, bit-identical, generating only the blocks they touch
    (each rank of a sharded run builds just its own shard)."""
    inst = instrument(cfg)
    conc = concentrations(cfg)
    dtype = np.float64 if cfg.dtype == "f64" else np.float32
    b0, b1 = r0 // BLOCK_ROWS, (max(r1, r0 + 1) - 1) // BLOCK_ROWS + 1
    tmp = np.empty(((b1 - b0) * BLOCK_ROWS, cfg.n_freq), dtype=dtype)
    view = _OffsetRows(tmp, b0 * BLOCK_ROWS)
    blocks = [b for b in range(b0, b1) if b * BLOCK_ROWS < cfg.n_pixels]
    threads = threads or min(len(blocks), max(1, len(os.sched_getaffinity(0))))
    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(lambda b: _block(cfg, inst, conc, b, view, dtype), blocks))
    off = r0 - b0 * BLOCK_ROWS
    return np.ascontiguousarray(tmp[off:off + (r1 - r0)]), reference(cfg, inst).astype(dtype), inst.omega


class _OffsetRows:
    def __init__(self, arr, base):
        self.arr, self.base = arr, base

    def __setitem__(self, sl, val):
        self.arr[sl.start - self.base:sl.stop - self.base] = val


def truth_imag(cfg: CubeConfig, rows: np.ndarray | None = None) -> np.ndarray:
    """Ground truth Im{chi/chi_NR} = Im{chi_R / chi_NR} for the given pixel rows."""
    inst = instrument(cfg)
    conc = concentrations(cfg)
    if rows is not None:
        conc = conc[rows]
    chi_r = conc @ inst.chi_species
    return (chi_r / inst.chi_nr[None, :]).imag


def lorentzian_spectrum(omega, centre, hwhm, amp, chi_nr=1.0):
    """chi = chi_nr + amp/(centre - omega - i hwhm): one complex Lorentzian."""
    return chi_nr + amp / (centre - omega - 1j * hwhm)


# ------------------------------------------------------------------------------------------------
# The paper's simulation workload (Fig. 2).  Physics of the
# measurement only (Eq. 1 with C_st = 1): a noiseless 3-chemical mixture of complex
# Lorentzian Raman spectra (22, 25, 10 peaks in 500-1700 cm^-1), real quadratic chi_nr per chemical
# with non-negative coefficients, a real linear chi_ref surrogate, sampled over -500..2500 cm^-1.
# Readings (A30): 812 channels at the paper's spacing (810 samples, rounded up to a multiple
# of 4 for the 16-B rows; omega_max = 2500 + 2 x 3000/809); the concentration map (Fig. 2(a), not in
# the text) = three smooth random fields normalised per pixel to a ternary mixture; peak amplitudes
# U(0.05, 0.5), HWHM U(4, 15) cm^-1; chi_nr,c = c0 + c1 x + c2 x^2, c ~ U(0.2, 1) (c0) / U(0, 1),
# x = (omega + 500)/3000; chi_ref = a + b x, a ~ U(0.5, 1), b ~ U(0, 0.5).
# ------------------------------------------------------------------------------------------------
SIM_BASE = (74, 246)
SIM_PEAKS = (22, 25, 10)
SIM_M = 812


def paper_sim_shape(scale: float) -> tuple[int, int]:
    return int(round(SIM_BASE[0] * scale)), int(round(SIM_BASE[1] * scale))


def paper_simulation(scale: float = 1.0, seed: int = 0):
    """Returns (I [N x 812] f32, I_ref [812] f32, truth Im{chi/chi_nr} [N x 812] f64, omega [812])."""
    H, W = paper_sim_shape(scale)
    g = _rng(seed, _STREAM_INSTRUMENT, 7)
    d = 3000.0 / 809.0
    w = -500.0 + d * np.arange(SIM_M)
    x = (w + 500.0) / 3000.0
    chi_r = np.zeros((3, SIM_M), dtype=np.complex128)
    for c, npk in enumerate(SIM_PEAKS):
        cen = g.uniform(500.0, 1700.0, npk)
        wid = g.uniform(4.0, 15.0, npk)
        amp = g.uniform(0.05, 0.5, npk)
        chi_r[c] = np.sum((amp * wid)[:, None] / (cen[:, None] - w[None, :] - 1j * wid[:, None]), axis=0)
    co = np.stack([g.uniform(0.2, 1.0, 3), g.uniform(0.0, 1.0, 3), g.uniform(0.0, 1.0, 3)], axis=1)
    chi_nr = co[:, 0:1] + co[:, 1:2] * x[None, :] + co[:, 2:3] * x[None, :] ** 2      # 3 x M, real > 0
    a, b = g.uniform(0.5, 1.0), g.uniform(0.0, 0.5)
    chi_ref = a + b * x
    # concentration map: three smooth fields on the unit square (the same map at every scale)
    gf = _rng(seed, _STREAM_FIELDS, 7)
    yy = (np.arange(H) + 0.5)[:, None] / H
    xx = (np.arange(W) + 0.5)[None, :] / W
    fields = np.empty((3, H * W))
    for c in range(3):
        fld = np.zeros((H, W))
        for _ in range(3):
            cy, cx, s = gf.uniform(0, 1), gf.uniform(0, 1), gf.uniform(0.1, 0.35)
            fld += np.exp(-((yy - cy) ** 2 + ((xx - cx) * W / H / 3.0) ** 2) / (2 * s * s))
        fields[c] = fld.ravel() + 0.05
    conc = (fields / fields.sum(axis=0, keepdims=True)).T                               # N x 3, sums to 1
    chi = conc @ (chi_r + chi_nr)                                                        # N x M
    nr = conc @ chi_nr                                                                   # N x M, real
    I = np.abs(chi) ** 2
    truth = (chi / nr).imag
    return I.astype(np.float32), (chi_ref ** 2).astype(np.float32), truth, w
