"""CPU tests of the C-ABI library: it loads, exports every function include/fkk.h declares, and its
host-only logic (eigensolver, shard ranges, extreme merging) is right -- including a 2-rank gloo run
of the sharded q selection (the multi-GPU exchange logic) on CPU."""
import os
import re

import numpy as np
import pytest

from oracle import fkk_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fkk():
    from paper_2005_07132_b200 import fkk
    return fkk


def test_library_exports_every_header_function():
    fkk = _fkk()
    hdr = open(os.path.join(ROOT, "include", "fkk.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"^\s*(?:fkk_status|void|const char\*|size_t|int32_t|int64_t)\s+\**\s*(\w+)\s*\(", hdr, re.M))
    assert len(names) >= 25
    for n in names:
        assert hasattr(fkk._lib, n), n
    assert names == set(fkk.EXPORTS)


def test_plan_create_rejects_bad_desc_without_gpu():
    fkk = _fkk()
    with pytest.raises(fkk.FkkError) as e:
        fkk.Plan(n_freq=30, rank_k=4, max_rows=10)        # M % 4 != 0
    assert e.value.name == "FKK_ERR_INVALID_ARG"
    with pytest.raises(fkk.FkkError) as e:
        fkk.Plan(n_freq=64, rank_k=100, max_rows=10)      # k > M
    assert e.value.name == "FKK_ERR_INVALID_ARG"
    with pytest.raises(fkk.FkkError) as e:
        fkk.Plan(n_freq=64, rank_k=4, max_rows=10, ratio_floor=1e-40)   # below FLT_MIN (fp32 log clamp)
    assert e.value.name == "FKK_ERR_INVALID_ARG"


@pytest.mark.parametrize("M,k", [(40, 7), (256, 30), (512, 12)])
def test_host_eig_matches_lapack(M, k):
    fkk = _fkk()
    rng = np.random.default_rng(M)
    A = rng.standard_normal((2 * M, M)) * np.exp(-np.arange(M) / 20.0)[None, :]
    G = A.T @ A
    V, lam = fkk.fkk_host_eig_topk(G, k)
    Vr, s, lr = O.eig_topk(G, k)
    assert np.max(np.abs(lam - lr[:k])) / lr[0] < 1e-13
    assert np.linalg.norm(V @ V.T - Vr @ Vr.T, 2) < 1e-10
    assert np.max(np.abs(V.T @ V - np.eye(k))) < 1e-12
    assert np.max(np.abs(V - Vr)) < 1e-9                   # same sign rule


def test_host_eig_on_log_ratio_gram_with_noise_plateau():
    """Clustered spectrum (noise plateau right at the cut), the situation of SURVEY finding 6."""
    fkk = _fkk()
    from synth import CONFIGS, generate
    I, Iref, _ = generate(CONFIGS["cfg1"])
    A = O.log_ratio(I, Iref, O.Params())
    G = A.T @ A
    k = 12
    V, lam = fkk.fkk_host_eig_topk(G, k)
    Vr, s, lr = O.eig_topk(G, k)
    assert np.max(np.abs(lam - lr[:k])) / lr[0] < 1e-12
    gap = (lr[k - 1] - lr[k]) / lr[0]
    assert np.linalg.norm(V @ V.T - Vr @ Vr.T, 2) < 1e-12 / gap + 1e-10


def test_shard_range_partition():
    fkk = _fkk()
    for n, w in [(10, 3), (703026, 8), (5, 8), (0, 2)]:
        rs = [fkk.fkk_shard_range(n, w, r) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def test_merge_extremes_ties_and_union():
    fkk = _fkk()
    # 2 ranks, k=2: col0 max tie (5.0 at global 7 and 3) -> 3; min at 9. col1 max 2 at 3, min -1 at 1
    vals = np.array([[[5.0, 0.0], [1.0, -1.0]], [[5.0, -2.0], [2.0, 0.5]]], dtype=np.float32)
    idx = np.array([[[7, 2], [0, 1]], [[3, 9], [3, 4]]], dtype=np.int64)
    q = fkk.fkk_merge_extremes(vals, idx, 2)
    assert list(q) == [1, 3, 9]


def _gloo_worker(rank, world, port, q_out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_07132_b200 import fkk
    from synth import CONFIGS, generate
    cfg = CONFIGS["cfg1"]
    I, Iref, _ = generate(cfg)
    A = O.log_ratio(I, Iref, O.Params())
    r0, r1 = fkk.fkk_shard_range(A.shape[0], world, rank)
    # the exchange steps of the sharded path: all-reduce of the Gram partials ...
    G = torch.from_numpy(A[r0:r1].T @ A[r0:r1])
    dist.all_reduce(G)
    V, lam = fkk.fkk_host_eig_topk(G.numpy(), cfg.rank_k)
    # ... and all-gather of the per-column (value, global index) extremes
    US = A[r0:r1] @ V
    vals = np.stack([US.max(0), US.min(0)], axis=1).astype(np.float32)
    idx = np.stack([US.argmax(0), US.argmin(0)], axis=1).astype(np.int64) + r0
    tv = [torch.zeros(cfg.rank_k, 2) for _ in range(world)]
    ti = [torch.zeros(cfg.rank_k, 2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(tv, torch.from_numpy(vals))
    dist.all_gather(ti, torch.from_numpy(idx))
    q = fkk.fkk_merge_extremes(np.stack([t.numpy() for t in tv]), np.stack([t.numpy() for t in ti]), cfg.rank_k)
    if rank == 0:
        q_out.put((q, G.numpy(), V))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_q_matches_single_process():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, qq)) for r in range(2)]
    for p in ps:
        p.start()
    q, G, V = qq.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    from synth import CONFIGS, generate
    cfg = CONFIGS["cfg1"]
    I, Iref, _ = generate(cfg)
    A = O.log_ratio(I, Iref, O.Params())
    assert np.max(np.abs(G - A.T @ A)) / np.max(np.abs(G)) < 1e-13
    assert list(q) == list(O.select_q(A @ V))


def test_library_has_no_undefined_internal_symbols():
    """Every fkk:: function the C-ABI library calls is defined in it (a shared library links with
    undefined symbols and would only fail when the call is made)."""
    import shutil
    import subprocess
    from paper_2005_07132_b200 import build as b
    if shutil.which("nm") is None:
        import pytest
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--undefined-only", b.LIB], capture_output=True, text=True).stdout
    bad = [ln for ln in out.splitlines() if ln.split()[0] == "U" and "fkk" in ln]
    assert not bad, bad
