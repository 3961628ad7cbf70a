"""GPU eigensolver (F4: the truncated SVD through G = A^T A) on synthetic symmetric
matrices through the C-ABI test hook fkk_debug_eig_topk.

Checked against what the mathematics fixes, at any size: LAPACK eigenvalues (numpy.linalg.eigvalsh,
the library routine the oracle's eig_topk step uses), the residual ||G V - V diag(lam)||, the
orthonormality of V and the sign rule (largest-|.| entry positive).  Both tridiagonalisation paths
are covered: row-resident in shared memory (M <= ~1800 on 148 SMs) and L2-streaming (larger M).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fkk(cuda_ok):
    from paper_2005_07132_b200 import fkk
    return fkk


def _spd_with_spectrum(lam, seed):
    rng = np.random.default_rng(seed)
    M = len(lam)
    Q, _ = np.linalg.qr(rng.standard_normal((M, M)))
    G = (Q * lam[None, :]) @ Q.T
    return 0.5 * (G + G.T)


def _check(fkk, G, k, *, tol_lam=1e-12, tol_res=1e-10):
    import torch
    V, lam = fkk.fkk_debug_eig_topk(torch.from_numpy(np.ascontiguousarray(G)).cuda(), k)
    V, lam = V.cpu().numpy(), lam.cpu().numpy()
    ref = np.linalg.eigvalsh(G)[::-1][:k]
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(lam - ref)) <= tol_lam * scale, np.max(np.abs(lam - ref)) / scale
    assert np.max(np.abs(G @ V - V * lam[None, :])) <= tol_res * scale
    assert np.max(np.abs(V.T @ V - np.eye(k))) <= 1e-10
    idx = np.argmax(np.abs(V), axis=0)
    assert np.all(V[idx, np.arange(k)] > 0)
    return V, lam


@pytest.mark.parametrize("M,k", [(4, 2), (37, 5), (300, 40), (1000, 60), (1600, 100)])
def test_eig_decaying_spectrum(fkk, M, k):
    lam = np.concatenate([np.geomspace(1e4, 1.0, min(M, 16)), np.linspace(0.9, 0.5, M - min(M, 16))])
    G = _spd_with_spectrum(lam, seed=M)
    _check(fkk, G, k)


def test_eig_paths(fkk):
    assert fkk.fkk_debug_eig_path(1000) == 1
    assert fkk.fkk_debug_eig_path(2400) == 0


def test_eig_l2_streaming_path(fkk):
    M, k = 2400, 24
    lam = np.concatenate([np.geomspace(1e3, 1.0, 12), np.linspace(0.8, 0.1, M - 12)])
    _check(fkk, _spd_with_spectrum(lam, seed=7), k)


def test_eig_noise_plateau_clusters(fkk):
    """A signal block above a dense plateau with relative gaps ~1e-7 and exact ties: the vectors
    inside a cluster are not unique, but the residual and orthonormality must still hold."""
    M, k = 512, 48
    plateau = 1.0 + 1e-7 * np.arange(M - 8)
    plateau[:6] = 1.0     # exact ties
    lam = np.concatenate([np.geomspace(50.0, 2.0, 8), plateau])
    _check(fkk, _spd_with_spectrum(lam, seed=3), k, tol_res=1e-10)


def test_eig_gram_of_log_ratio(fkk):
    """The matrix the path actually solves: the Gram of a cfg1-generator log-ratio cube (fp64)."""
    from oracle import fkk_oracle as O
    from synth import CONFIGS, generate
    I, Iref, _ = generate(CONFIGS["cfg1"])
    G = O.gram(O.log_ratio(I, Iref, O.Params()))
    _check(fkk, G, 12)


def test_eig_rank_deficient(fkk):
    """Exact zero eigenvalues below the kept rank (tau = 0 reflectors, zero Sturm pivots)."""
    M, k = 64, 8
    rng = np.random.default_rng(5)
    B = rng.standard_normal((M, 5))
    G = B @ B.T
    _check(fkk, G, k, tol_lam=1e-11)
