"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on the same seeded cubes.

Tolerances (BASELINE.json north_star):
  direct KK           max_n ||K_gpu - K_or||_inf / ||K_or||_inf <= 1e-5
  factorized, stages  G, US max-norm relative <= 1e-5; |d s_i| <= 1e-5 s_1 (Weyl);
                      F6..F11 from the GPU's (V, s, q): Im K <= 1e-4
  factorized, e2e     max|Im K_gpu - Im K_or| / max|Im K_or| <= 1e-3 (q must agree)
"""
import numpy as np
import pytest

from oracle import fkk_oracle as O
from synth import CONFIGS, generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda(cuda_ok):
    import torch
    return torch


@pytest.fixture(scope="module")
def fkk():
    from paper_2005_07132_b200 import fkk
    return fkk


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rel_inf(K, R):
    return np.max(np.max(np.abs(K - R), axis=1) / np.max(np.abs(R), axis=1))


@pytest.fixture(scope="module")
def cfg1():
    I, Iref, _ = generate(CONFIGS["cfg1"])
    return I, Iref


# ------------------------------------------------------------------------- direct path -----------
@pytest.mark.parametrize("pad", ["reflect", "zero"])
@pytest.mark.parametrize("rows", [1, 33, 301])
def test_direct_cfg1_f64_input(torch_cuda, fkk, cfg1, pad, rows):
    I, Iref = cfg1
    I = I[:rows]
    p = O.Params(pad=pad)
    K_or = O.kk_direct(I, Iref, p)
    plan = fkk.Plan(512, 12, rows, pad=pad, in_dtype="f64")
    K = plan.direct(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    assert _rel_inf(K, K_or) <= 1e-5


@pytest.mark.parametrize("rows", [1, 33, 301])
def test_direct_cfg1_f32_input_odd_rows(torch_cuda, fkk, cfg1, rows):
    """fp32 input takes direct_finish's prefetch pipeline (next pair's phi_err rows bulk-copied into a
    staging buffer, a lone last row without a partner): odd row counts, 1e-5 against the oracle run on
    the same fp32 values."""
    I, Iref = cfg1
    I32 = I[:rows].astype(np.float32)
    R32 = Iref.astype(np.float32)
    K_or = O.kk_direct(I32.astype(np.float64), R32.astype(np.float64), O.Params())
    plan = fkk.Plan(512, 12, rows, in_dtype="f32")
    K = plan.direct(_dev(torch_cuda, I32), _dev(torch_cuda, R32)).cpu().numpy()
    assert _rel_inf(K, K_or) <= 1e-5


def test_direct_cfg2_sample_f32(torch_cuda, fkk):
    I, Iref, _ = generate(CONFIGS["cfg2"])
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(I.shape[0], 200, replace=False))
    plan = fkk.Plan(1000, 40, I.shape[0])
    K = plan.direct(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    K_or = O.kk_direct(I[rows].astype(np.float64), Iref.astype(np.float64), O.Params())
    assert _rel_inf(K[rows], K_or) <= 1e-5
    # imag-only layout gives the same Im part
    plan_i = fkk.Plan(1000, 40, 4096, imag_only=True)
    Ki = plan_i.direct(_dev(torch_cuda, I[:4096]), _dev(torch_cuda, Iref)).cpu().numpy()
    assert np.array_equal(Ki, K[:4096].imag)


@pytest.mark.parametrize("M", [16, 100, 132, 1020, 1600, 2048])
def test_direct_segment_edge_sizes(torch_cuda, fkk, M):
    """The warp-partitioned ALS splits M into P = ceil(M/T) segments of T = max(4, ceil(M/32)) rows and
    extends the last one with zero-weight rows (reading A31): M = 16 (4 segments of 4 rows, 2-row
    interiors), 100 (25 x 4, no padding), 132 (27 x 5, 3 padding rows), 1020 (32 x 32, 4 rows),
    1600 (32 x 50, the cfg4 channel count), 2048 (64-row segments: 62-bit interior masks; L = 4096, the
    largest direct-path FFT)."""
    cfg = CONFIGS["cfg1"].with_(height=4, width=9, n_freq=M)
    I, Iref, _ = generate(cfg)
    K_or = O.kk_direct(I, Iref, O.Params())
    plan = fkk.Plan(M, 4, I.shape[0], in_dtype="f64")
    K = plan.direct(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    assert _rel_inf(K, K_or) <= 1e-5


def test_direct_passthrough_and_scale(torch_cuda, fkk):
    rng = np.random.default_rng(1)
    Iref = rng.uniform(0.5, 1.5, 1000).astype(np.float32)
    I = np.stack([Iref, 2.5 * Iref]).astype(np.float32)
    plan = fkk.Plan(1000, 8, 2)
    K = plan.direct(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    assert np.max(np.abs(K - 1.0)) < 1e-5


def test_errors_reported(torch_cuda, fkk, cfg1):
    I, Iref = cfg1
    plan = fkk.Plan(512, 12, 64, in_dtype="f64")
    bad = Iref.copy()
    bad[7] = -1.0
    with pytest.raises(fkk.FkkError) as e:
        plan.transform(_dev(torch_cuda, I[:64]), _dev(torch_cuda, bad))
    assert e.value.name == "FKK_ERR_BAD_REFERENCE"
    In = I[:64].copy()
    In[3, 5] = np.nan
    with pytest.raises(fkk.FkkError) as e:
        plan.transform(_dev(torch_cuda, In), _dev(torch_cuda, Iref))
    assert e.value.name == "FKK_ERR_NONFINITE_INPUT"
    # the plan stays usable after an error
    plan.transform(_dev(torch_cuda, I[:64]), _dev(torch_cuda, Iref))


# ------------------------------------------------------------------------- factorized path -------
GEMMS = ["3xtf32", "fp32_simt"]


def _factorized_check(torch, fkk, I, Iref, k, *, e2e_tol=1e-3, loopback=0, in_dtype="f32", gemm=None):
    p = O.Params()
    plan = fkk.Plan(I.shape[1], k, I.shape[0], in_dtype=in_dtype, loopback_shards=loopback, gemm=gemm)
    Id, Rd = _dev(torch, I), _dev(torch, Iref)
    K = plan.transform(Id, Rd).cpu().numpy()
    G_gpu, s_gpu, V_gpu, US_gpu = plan.stage("G"), plan.stage("S"), plan.stage("V"), plan.stage("US")
    q_gpu = plan.stage("Q")
    A = O.log_ratio(I, Iref, p)
    # stage-wise: Gram, singular values, projection with the GPU's V
    G_or = O.gram(A)
    assert np.max(np.abs(G_gpu - G_or)) / np.max(np.abs(G_or)) <= 1e-5
    V_or, s_or, lam = O.eig_topk(G_or, k)
    # Weyl: |d sigma_i| <= ||dA||_2, a normwise bound -> relative to sigma_1 (DESIGN.md parity contract)
    assert np.max(np.abs(s_gpu - s_or)) / s_or[0] <= 1e-5
    # the GPU eigensolver on the GPU's own G: residual and orthonormality (property at any size)
    lam_gpu = s_gpu ** 2
    assert np.max(np.abs(G_gpu @ V_gpu - V_gpu * lam_gpu[None, :])) / lam_gpu[0] <= 1e-10
    assert np.max(np.abs(V_gpu.T @ V_gpu - np.eye(k))) <= 1e-10
    US_ref = A @ V_gpu
    assert np.max(np.abs(US_gpu - US_ref)) / np.max(np.abs(US_ref)) <= 1e-5
    gap = (lam[k - 1] - lam[k]) / lam[k - 1]
    # F6..F11 from the GPU's (V, s, q): the oracle on the same inputs
    V32 = V_gpu.astype(np.float32).astype(np.float64)
    out_from = O.fkk_ec_from(I, Iref, V32, s_gpu, q_gpu, p)
    K_from = plan.transform_from(Id, Rd, _dev(torch, np.ascontiguousarray(V32.T.astype(np.float32))), s_gpu,
                                 q_gpu).cpu().numpy()
    im_err_from = np.max(np.abs(K_from.imag - out_from["K"].imag)) / np.max(np.abs(out_from["K"].imag))
    assert im_err_from <= 1e-4, im_err_from
    # end to end
    out = O.fkk_ec(I, Iref, k, p)
    same_q = np.array_equal(out["q"], q_gpu)
    im_err = np.max(np.abs(K.imag - out["K"].imag)) / np.max(np.abs(out["K"].imag))
    diag = dict(gap=gap, same_q=same_q, im_err=im_err, im_err_from=im_err_from)
    assert same_q, diag
    assert im_err <= e2e_tol, diag
    return plan, K, diag


@pytest.mark.parametrize("gemm", GEMMS)
def test_factorized_cfg1(torch_cuda, fkk, cfg1, gemm):
    I, Iref = cfg1
    _factorized_check(torch_cuda, fkk, I, Iref, 12, in_dtype="f64", gemm=gemm)


@pytest.mark.parametrize("gemm", GEMMS)
def test_factorized_cfg1_loopback_shards_invariant(torch_cuda, fkk, cfg1, gemm):
    I, Iref = cfg1
    plan1, K1, _ = _factorized_check(torch_cuda, fkk, I, Iref, 12, in_dtype="f64", gemm=gemm)
    plan3, K3, _ = _factorized_check(torch_cuda, fkk, I, Iref, 12, in_dtype="f64", loopback=3, gemm=gemm)
    assert np.array_equal(plan1.stage("Q"), plan3.stage("Q"))
    assert np.max(np.abs(K1 - K3)) / np.max(np.abs(K1)) < 1e-4


@pytest.mark.parametrize("gemm", GEMMS)
def test_factorized_ragged_small(torch_cuda, fkk, cfg1, gemm):
    I, Iref = cfg1
    _factorized_check(torch_cuda, fkk, I[:777], Iref, 12, in_dtype="f64", gemm=gemm)


@pytest.fixture(scope="module")
def cfg2():
    I, Iref, _ = generate(CONFIGS["cfg2"])
    return I, Iref


@pytest.mark.parametrize("gemm", GEMMS)
def test_factorized_cfg2(torch_cuda, fkk, cfg2, gemm):
    I, Iref = cfg2
    _factorized_check(torch_cuda, fkk, I, Iref, 40, gemm=gemm)


def test_projection_repeatable_multi_tile(torch_cuda, fkk, cfg2):
    """US = A0 V on the tensor cores (TMA + TMEM-A pipeline) against float64 A0 V, repeated: every CTA
    walks several tiles with its rings and accumulator sets wrapping, so an early slot release (a
    pipeline race) shows up as scattered wrong rows after the first tile."""
    I, Iref = cfg2
    A = O.log_ratio(I, Iref, O.Params())
    plan = fkk.Plan(1000, 40, I.shape[0])
    Id, Rd = _dev(torch_cuda, I), _dev(torch_cuda, Iref)
    for _ in range(3):
        plan.transform(Id, Rd)
        V, US = plan.stage("V"), plan.stage("US")
        ref = A @ V
        assert np.max(np.abs(US - ref)) / np.max(np.abs(ref)) <= 1e-5


def test_gram_tc_equals_simt_in_fp32_accuracy(torch_cuda, fkk, cfg2):
    """3xTF32 tcgen05 Gram vs the exact-fp32 CUDA-core Gram vs fp64 (max-norm relative)."""
    I, Iref = cfg2
    I = I[:20000]
    G = {}
    for g in GEMMS:
        plan = fkk.Plan(1000, 40, I.shape[0], gemm=g)
        plan.svd(_dev(torch_cuda, I), _dev(torch_cuda, Iref))
        G[g] = plan.stage("G")
    G_or = O.gram(O.log_ratio(I, Iref, O.Params()))
    for g in GEMMS:
        assert np.max(np.abs(G[g] - G_or)) / np.max(np.abs(G_or)) <= 2e-6, g


@pytest.mark.parametrize("mode", ["0", "1"])
def test_image_gram_variants(torch_cuda, fkk, cfg2, mode, monkeypatch):
    """Both pre-split-image Gram kernels (0: 1-CTA 128x128 tiles, 1: CTA pairs 256x256, the default at
    M = 1000) against the fp64 oracle Gram, at a pixel count that leaves ragged stages and splits."""
    monkeypatch.setenv("FKK_GRAM_MODE", mode)
    I, Iref = cfg2
    I = I[:30001]
    plan = fkk.Plan(1000, 40, I.shape[0])
    plan.svd(_dev(torch_cuda, I), _dev(torch_cuda, Iref))
    G_or = O.gram(O.log_ratio(I, Iref, O.Params()))
    assert np.max(np.abs(plan.stage("G") - G_or)) / np.max(np.abs(G_or)) <= 2e-6


def test_factorized_odd_channel_blocks(torch_cuda, fkk, cfg2):
    """M = 640 (five 128-channel blocks: the 1-CTA image Gram is the default there) end to end."""
    I, Iref = cfg2
    _factorized_check(torch_cuda, fkk, np.ascontiguousarray(I[:20000, :640]), np.ascontiguousarray(Iref[:640]), 40)


# ------------------------------------------------------- conventional workflow (NEXT 2) ----------
@pytest.mark.parametrize("k_keep", [6, 12])
def test_conventional_svd_denoise_cfg1(torch_cuda, fkk, cfg1, k_keep):
    """fkk_conventional (rank-k SVD denoise of the raw cube, then direct KK) against the oracle's
    conventional_workflow on the same cube: the denoised cube goes through the fp32 tensor-core SVD, so
    the bar is the factorized path's (1e-3 max-norm relative, Im and Re)."""
    I, Iref = cfg1
    I32 = I[:1024].astype(np.float32)   # (the oracle's per-spectrum ALS bounds the size)
    plan = fkk.Plan(I.shape[1], 12, I32.shape[0], in_dtype="f32")
    K = plan.conventional(_dev(torch_cuda, I32), _dev(torch_cuda, Iref.astype(np.float32)), k_keep).cpu().numpy()
    K_or = O.conventional_workflow(I32.astype(np.float64), Iref.astype(np.float32).astype(np.float64), k_keep)
    err = np.max(np.abs(K - K_or)) / np.max(np.abs(K_or))
    print(f"conventional cfg1 k={k_keep}: {err:.3e}")
    assert err <= 1e-3, err


@pytest.mark.parametrize("rows,k_keep", [(1, 1), (33, 3), (200, 12)])
def test_conventional_ragged_small(torch_cuda, fkk, cfg1, rows, k_keep):
    """Ragged / tiny cubes through the conventional workflow (one Gram split, partial tiles)."""
    I, Iref = cfg1
    I32 = I[:rows].astype(np.float32)
    R32 = Iref.astype(np.float32)
    plan = fkk.Plan(I.shape[1], 12, rows, in_dtype="f32")
    K = plan.conventional(_dev(torch_cuda, I32), _dev(torch_cuda, R32), k_keep).cpu().numpy()
    K_or = O.conventional_workflow(I32.astype(np.float64), R32.astype(np.float64), k_keep)
    err = np.max(np.abs(K - K_or)) / np.max(np.abs(K_or))
    assert err <= 1e-3, err


def test_conventional_cfg2_sample(torch_cuda, fkk, cfg2):
    I, Iref = cfg2
    I = I[:512]
    plan = fkk.Plan(1000, 40, I.shape[0])
    K = plan.conventional(_dev(torch_cuda, I), _dev(torch_cuda, Iref), 20).cpu().numpy()
    K_or = O.conventional_workflow(I.astype(np.float64), Iref.astype(np.float64), 20)
    err = np.max(np.abs(K - K_or)) / np.max(np.abs(K_or))
    print(f"conventional cfg2 k=20: {err:.3e}")
    assert err <= 1e-3, err


# ------------------------------------------------------------------------- ML reuse --------------
def test_ml_apply_matches_oracle_and_self_consistent(torch_cuda, fkk):
    cfg = CONFIGS["cfg5_train"].with_(height=64, width=64)
    I, Iref, _ = generate(cfg)
    Ia, _, _ = generate(CONFIGS["cfg5_apply"].with_(height=48, width=40))
    k = 20
    plan = fkk.Plan(1000, k, I.shape[0])
    K_train, basis = plan.transform(_dev(torch_cuda, I), _dev(torch_cuda, Iref), return_basis=True)
    # oracle model from the GPU's V, s, q (stage-wise) and apply on the new cube
    V = plan.stage("V").astype(np.float32).astype(np.float64)
    s = plan.stage("S")
    q = plan.stage("Q")
    p = O.Params()
    out = O.fkk_ec_from(I, Iref, V, s, q, p)
    model = dict(f=out["f"], W=O.ml_projector(V, s, p), B_amp=out["B_amp"], B_ph=out["B_ph"])
    Ka = plan.apply(basis, _dev(torch_cuda, Ia)).cpu().numpy()
    Ka_or = O.ml_apply(Ia.astype(np.float64), Iref.astype(np.float64), model, p)
    assert np.max(np.abs(Ka.imag - Ka_or.imag)) / np.max(np.abs(Ka_or.imag)) <= 1e-4
    # lambda_ml = 0: applying to the training cube reproduces the training output (P14)
    Kt = plan.apply(basis, _dev(torch_cuda, I)).cpu().numpy()
    assert np.max(np.abs(Kt - K_train.cpu().numpy())) / np.max(np.abs(Kt)) <= 1e-4
    assert basis.info() == dict(n_freq=1000, rank_k=k, fft_len=2048)
    # incompatible basis
    plan2 = fkk.Plan(512, 12, 10)
    with pytest.raises(fkk.FkkError) as e:
        plan2.apply(basis, _dev(torch_cuda, np.ones((4, 512), np.float32)))
    assert e.value.name == "FKK_ERR_INCOMPATIBLE_BASIS"


def test_host_buffer_variants(torch_cuda, fkk, cfg1):
    I, Iref = cfg1
    plan = fkk.Plan(512, 12, I.shape[0], in_dtype="f64")
    K_dev = plan.direct(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    out = np.empty((I.shape[0], 512), np.complex64)
    plan.direct_host(I, Iref, out)
    assert np.array_equal(out, K_dev)
    Kt_dev = plan.transform(_dev(torch_cuda, I), _dev(torch_cuda, Iref)).cpu().numpy()
    plan.transform_host(I, Iref, out)
    assert np.max(np.abs(out - Kt_dev)) <= 1e-6 * np.max(np.abs(Kt_dev))


def test_transform_host_stream_matches_per_cube_calls(torch_cuda, fkk, cfg1):
    """fkk_transform_host_stream: three different host cubes through the copy/compute pipeline, each
    equal to its own fkk_transform_host; an output buffer reused with stride 2 holds the later cube."""
    I, Iref = cfg1
    rng = np.random.default_rng(5)
    cubes = [np.ascontiguousarray(I * s * np.exp(0.05 * rng.standard_normal(I.shape))) for s in (1.0, 1.7, 0.6)]
    plan = fkk.Plan(512, 12, I.shape[0], in_dtype="f64")
    ref = []
    for c in cubes:
        o = np.empty((I.shape[0], 512), np.complex64)
        plan.transform_host(c, Iref, o)
        ref.append(o)
    outs = [np.empty((I.shape[0], 512), np.complex64) for _ in range(3)]
    ms = plan.transform_host_stream(cubes, Iref, outs)
    assert ms.shape == (3,) and np.all(ms > 0)
    for o, r in zip(outs, ref):
        assert np.max(np.abs(o - r)) <= 1e-6 * np.max(np.abs(r))
    shared = [outs[0], outs[1], outs[0]]
    plan.transform_host_stream(cubes, Iref, shared)
    assert np.max(np.abs(outs[0] - ref[2])) <= 1e-6 * np.max(np.abs(ref[2]))
    assert np.max(np.abs(outs[1] - ref[1])) <= 1e-6 * np.max(np.abs(ref[1]))


def test_q_ties_take_the_lowest_pixel(torch_cuda, fkk, cfg2):
    """Every spectrum duplicated (rows 2i and 2i+1 equal, in the same projection tile): each column
    extreme of US ties between two pixels, and q (Eqs. 13-15, ties -> lowest pixel, reading A12) must
    hold only even pixels and equal the oracle's q on the same cube."""
    I, Iref = cfg2
    Id2 = np.repeat(I[:6000], 2, axis=0)
    plan = fkk.Plan(1000, 40, Id2.shape[0])
    plan.transform(_dev(torch_cuda, Id2), _dev(torch_cuda, Iref))
    q = plan.stage("Q")
    US = plan.stage("US")
    assert np.array_equal(US[0::2], US[1::2])          # the duplicated rows project bit-identically
    assert np.all(q % 2 == 0), q
    out = O.fkk_ec(Id2.astype(np.float64), Iref.astype(np.float64), 40, O.Params())
    assert np.array_equal(q, out["q"])


def test_nccl_backend_one_rank(torch_cuda, fkk, cfg2):
    """The NCCL collective backend (dlopen'ed libnccl, ncclCommInitRank, the row-count / extremes
    all-gathers, the Gram and X all-reduces, the flags max-reduce and the deadline-polled syncs) over a
    1-rank communicator on this GPU: the same results as the local backend, errors still reported and
    the plan reusable, for the Gram and the range-finder SVD."""
    I, Iref = cfg2
    I = I[:20000]
    Id, Rd = _dev(torch_cuda, I), _dev(torch_cuda, Iref)
    for svd in ("gram", "range_finder"):
        loc = fkk.Plan(1000, 40, I.shape[0], svd=svd)
        nc = fkk.Plan(1000, 40, I.shape[0], svd=svd, world_size=1, rank=0, nccl_id=fkk.fkk_get_nccl_unique_id())
        K0 = loc.transform(Id, Rd).cpu().numpy()
        K1 = nc.transform(Id, Rd).cpu().numpy()
        assert np.array_equal(loc.stage("Q"), nc.stage("Q"))
        assert np.max(np.abs(K1 - K0)) <= 1e-6 * np.max(np.abs(K0))
        bad = I[:2000].copy()
        bad[3, 5] = np.nan
        with pytest.raises(fkk.FkkError) as e:
            nc.transform(_dev(torch_cuda, bad), Rd)
        assert e.value.name == "FKK_ERR_NONFINITE_INPUT"
        K2 = nc.transform(Id, Rd).cpu().numpy()
        assert np.max(np.abs(K2 - K0)) <= 1e-6 * np.max(np.abs(K0))
