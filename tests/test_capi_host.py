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


def _gloo_worker(rank, world, port, q_out, nan_rank):
    """One rank of the sharded transform's exchange sequence, run by the LIBRARY (fkk_exchange_selftest:
    the same C++ sequence functions the NCCL path calls) over gloo collectives on CPU."""
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
    k = cfg.rank_k
    # uneven shards: rank r owns a contiguous block of 1000 + 1000 r rows (the global offsets come from
    # the library's row-count allgather, not from here)
    sizes = [1000 + 1000 * r for r in range(world)]
    r0 = sum(sizes[:rank])
    Al = A[r0:r0 + sizes[rank]]

    def allgather(b):
        out = [torch.zeros(b.size, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(b))
        return np.concatenate([o.numpy() for o in out])

    def allreduce_sum(a):
        t = torch.from_numpy(a)
        dist.all_reduce(t)
        return t.numpy()

    def allreduce_max(a):
        t = torch.from_numpy(a)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.numpy()

    # local inputs of the exchange: the Gram partial, and (after the eig of the global G, which every
    # rank computes identically) the local projection's column extremes with GLOBAL indices
    Gl = Al.T @ Al
    Gtot = torch.from_numpy(Gl.copy())
    dist.all_reduce(Gtot)
    V, lam = fkk.fkk_host_eig_topk(Gtot.numpy(), k)
    US = (Al @ V).astype(np.float32)
    vals = np.stack([US.max(0), US.min(0)], axis=1)[None]
    idx = (np.stack([US.argmax(0), US.argmin(0)], axis=1) + r0)[None]
    flags = 2 if rank == nan_rank else 0      # a non-finite value seen by one rank only
    res = fkk.fkk_exchange_selftest(world, rank, allgather, allreduce_sum, allreduce_max, Al.shape[0], A.shape[1], k,
                                    1, Gl, vals, idx, US, flags)
    if rank == 0:
        q_out.put((res, V))
    dist.destroy_process_group()


def test_two_rank_gloo_library_exchange_sequence():
    """The pixel-sharded exchange through the library's own sequence code on 2 gloo
    ranks with uneven shards: row offsets / global N from the row-count allgather, the all-reduced
    Gram equals the single-process Gram, q from the merged extremes equals the oracle's select_q, X =
    US[q] is the global one, and an error flag raised on ONE rank reaches every rank."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, qq, 1)) for r in range(2)]
    for p in ps:
        p.start()
    res, V = qq.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    from synth import CONFIGS, generate
    cfg = CONFIGS["cfg1"]
    I, Iref, _ = generate(cfg)
    A = O.log_ratio(I, Iref, O.Params())[:3000]
    assert res["row0"] == 0 and res["n_global"] == 3000
    assert np.max(np.abs(res["G"] - A.T @ A)) / np.max(np.abs(A.T @ A)) < 1e-13
    US = A @ V
    q = O.select_q(US.astype(np.float32))
    assert list(res["q"]) == list(q)
    assert np.max(np.abs(res["X"] - US.astype(np.float32)[q])) < 1e-6
    assert res["flags"] == 2


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


def test_range_finder_test_matrix_matches_oracle_generator():
    """The library's host generator of the range finder's Omega (SplitMix64 + Box-Muller) against the
    oracle's independent implementation (oracle.range_finder_omega, pinned to SplitMix64's reference
    vectors by P27): identical to the last bit or so (both fp64 libm)."""
    fkk = _fkk()
    M, l = 257, 13
    out = fkk.fkk_range_finder_omega(11, M, l)
    ref = O.range_finder_omega(11, M, l)
    assert np.max(np.abs(out - ref)) <= 1e-14
