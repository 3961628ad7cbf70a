"""Thin ctypes binding of the fKK-EC C-ABI (include/fkk.h).  Argument marshalling only: every
step of the method runs in libfkk.so (CUDA kernels + the C++ plan).  torch is used for device
memory and the current CUDA stream.  There is no fallback: if libfkk.so is missing or does not load,
importing this module raises.

Function names mirror the C-ABI: fkk_plan_create, fkk_svd, fkk_transform, fkk_transform_from,
fkk_apply_trained_basis, kk_direct_batch (+ *_host variants), fkk_get_stage, fkk_host_eig_topk,
fkk_shard_range, fkk_merge_extremes.  ``Plan`` wraps a plan handle with the same calls as methods.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FKK_LIB", os.path.join(_HERE, "lib", "libfkk.so"))
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libfkk.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ enums / status
FKK_OK = 0
STATUS = {0: "FKK_OK", 1: "FKK_ERR_INVALID_ARG", 2: "FKK_ERR_NONFINITE_INPUT", 3: "FKK_ERR_BAD_REFERENCE",
          4: "FKK_ERR_NUMERICAL", 5: "FKK_ERR_INCOMPATIBLE_BASIS", 6: "FKK_ERR_STATE", 7: "FKK_ERR_CUDA",
          8: "FKK_ERR_NCCL", 9: "FKK_ERR_OOM", 10: "FKK_ERR_NOT_IMPLEMENTED"}
PAD = {"reflect": 0, "zero": 1}
GEMM = {"3xtf32": 0, "fp32_simt": 1}
F_MODE = {"one": 0, "eq9": 1}
SVD_MODE = {"gram": 0, "range_finder": 1}
STAGES = {"G": 0, "S": 1, "V": 2, "US": 3, "Q": 4, "HV": 5, "PHI_ERR": 6, "PHI_PEC": 7, "V_SEC": 8, "B": 9,
          "LAMBDA": 10, "F": 11}


class FkkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("n_freq", ctypes.c_int32), ("max_rows", ctypes.c_int64), ("rank_k", ctypes.c_int32),
        ("fft_len", ctypes.c_int32), ("pad_mode", ctypes.c_int32), ("ratio_floor", ctypes.c_double),
        ("f_mode", ctypes.c_int32), ("f_alpha", ctypes.c_double), ("f_sigma_g", ctypes.c_double),
        ("als_lambda", ctypes.c_double), ("als_p", ctypes.c_double), ("als_iters", ctypes.c_int32),
        ("sg_window", ctypes.c_int32), ("sg_order", ctypes.c_int32), ("ridge_rel", ctypes.c_double),
        ("ml_ridge_rel", ctypes.c_double), ("gemm_impl", ctypes.c_int32), ("out_layout", ctypes.c_int32),
        ("in_dtype", ctypes.c_int32), ("device", ctypes.c_int32), ("world_size", ctypes.c_int32),
        ("rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("loopback_shards", ctypes.c_int32),
        ("svd_mode", ctypes.c_int32), ("rf_oversample", ctypes.c_int32), ("rf_power_iters", ctypes.c_int32),
        ("rf_seed", ctypes.c_uint64),
    ]


_vp, _i64, _i32, _dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)
_SIGS = {
    "fkk_plan_desc_init": (None, [ctypes.POINTER(PlanDesc), _i32, _i32, _i64]),
    "fkk_get_nccl_unique_id": (_i32, [ctypes.c_char_p]),
    "fkk_plan_create": (_i32, [ctypes.POINTER(PlanDesc), ctypes.POINTER(_vp)]),
    "fkk_plan_destroy": (_i32, [_vp]),
    "fkk_last_error": (ctypes.c_char_p, [_vp]),
    "fkk_plan_set_stream": (_i32, [_vp, _vp]),
    "fkk_plan_sync": (_i32, [_vp]),
    "fkk_svd": (_i32, [_vp, _vp, _i64, _vp, _vp, _dp]),
    "fkk_transform": (_i32, [_vp, _vp, _i64, _vp, _vp, ctypes.POINTER(_vp)]),
    "fkk_apply_trained_basis": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "kk_direct_batch": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "fkk_conventional": (_i32, [_vp, _vp, _i64, _vp, _i32, _vp]),
    "fkk_transform_host": (_i32, [_vp, _vp, _i64, _vp, _vp, ctypes.POINTER(_vp)]),
    "fkk_apply_trained_basis_host": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "fkk_transform_host_stream": (_i32, [_vp, ctypes.POINTER(_vp), _i32, _i64, _vp, ctypes.POINTER(_vp),
                                         ctypes.POINTER(ctypes.c_float)]),
    "kk_direct_batch_host": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "fkk_apply_trained_basis_stream": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, ctypes.POINTER(ctypes.c_float)]),
    "fkk_basis_destroy": (_i32, [_vp]),
    "fkk_basis_info": (_i32, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "fkk_stage_size": (ctypes.c_size_t, [_vp, _i32]),
    "fkk_get_stage": (_i32, [_vp, _i32, _vp, ctypes.c_size_t, _i32]),
    "fkk_transform_from": (_i32, [_vp, _vp, _i64, _vp, _vp, _dp, ctypes.POINTER(_i64), _i32, _vp]),
    "fkk_enable_timing": (_i32, [_vp, _i32]),
    "fkk_stage_times": (_i32, [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), _i32]),
    "fkk_last_launch_count": (_i64, [_vp]),
    "fkk_debug_als_solves": (_i64, [_vp]),
    "fkk_range_finder_omega": (_i32, [ctypes.c_uint64, _i32, _i32, _dp]),
    "fkk_exchange_selftest": (_i32, [_vp, _i64, _i32, _i32, _i32, _dp, ctypes.POINTER(ctypes.c_float),
                                     ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_i32),
                                     ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                     ctypes.POINTER(_i32), _dp]),
    "fkk_host_eig_topk": (_i32, [_dp, _i32, _i32, _dp, _dp]),
    "fkk_debug_tc_mma": (_i32, [_i32, _vp, _vp, _vp, _i32]),
    "fkk_debug_eig_topk": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "fkk_debug_eig_path": (_i32, [_i32]),
    "fkk_debug_tridiag": (_i32, [_vp, _i32, _vp]),
    "fkk_shard_range": (None, [_i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "fkk_merge_extremes": (_i32, [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_i64), _i32, _i32,
                                  ctypes.POINTER(_i64)]),
}
EXPORTS = tuple(_SIGS)
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(plan_handle, st: int):
    if st != FKK_OK:
        msg = _lib.fkk_last_error(plan_handle)
        raise FkkError(st, msg.decode() if msg else "")


def _torch():
    import torch
    return torch


def _dev_ptr(t, name: str):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


class Basis:
    """A trained ML:fKK-EC basis owned by the caller."""

    def __init__(self, handle):
        self._h = handle

    @property
    def handle(self):
        return self._h

    def info(self):
        m, k, L = _i32(), _i32(), _i32()
        _check(None, _lib.fkk_basis_info(self._h, ctypes.byref(m), ctypes.byref(k), ctypes.byref(L)))
        return dict(n_freq=m.value, rank_k=k.value, fft_len=L.value)

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fkk_basis_destroy(self._h)
        self._h = None

    __del__ = close


class Plan:
    """fkk_plan: workspace + stream for one device and one (M, k, max_rows)."""

    def __init__(self, n_freq: int, rank_k: int, max_rows: int, *, pad: str = "reflect", fft_len: int = 0,
                 ratio_floor: float = 1e-6, f_mode: str = "one", f_alpha: float = 0.0, f_sigma_g: float = 1.0,
                 als_lambda: float = 1e4, als_p: float = 1e-3, als_iters: int = 10, sg_window: int = 0,
                 ridge_rel: float = 1e-3, ml_ridge_rel: float = 0.0, gemm: str | None = None,
                 imag_only: bool = False, in_dtype: str = "f32", device: int = 0, world_size: int = 1,
                 rank: int = 0, nccl_id: bytes | None = None, loopback_shards: int = 0, timing: bool = False,
                 svd: str = "gram", rf_oversample: int = 10, rf_power_iters: int = 1, rf_seed: int = 0):
        d = PlanDesc()
        _lib.fkk_plan_desc_init(ctypes.byref(d), n_freq, rank_k, max_rows)
        d.fft_len = fft_len
        d.pad_mode = PAD[pad]
        d.ratio_floor = ratio_floor
        d.f_mode = F_MODE[f_mode]
        d.f_alpha, d.f_sigma_g = f_alpha, f_sigma_g
        d.als_lambda, d.als_p, d.als_iters = als_lambda, als_p, als_iters
        d.sg_window = sg_window
        d.ridge_rel, d.ml_ridge_rel = ridge_rel, ml_ridge_rel
        if gemm is not None:
            d.gemm_impl = GEMM[gemm]
        d.out_layout = 1 if imag_only else 0
        d.in_dtype = 1 if in_dtype == "f64" else 0
        d.device = device
        d.world_size, d.rank = world_size, rank
        self._nccl_buf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        d.nccl_id = ctypes.cast(self._nccl_buf, ctypes.c_void_p) if self._nccl_buf is not None else None
        d.loopback_shards = loopback_shards
        d.svd_mode = SVD_MODE[svd]
        d.rf_oversample, d.rf_power_iters, d.rf_seed = rf_oversample, rf_power_iters, rf_seed
        self.desc = d
        self.n_freq, self.rank_k, self.max_rows = n_freq, rank_k, max_rows
        self.imag_only = imag_only
        self.in_dtype = in_dtype
        self.device = device
        h = _vp()
        _check(None, _lib.fkk_plan_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        if timing:
            _lib.fkk_enable_timing(h, 1)

    # -------------------------------------------------------------- plumbing
    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fkk_plan_destroy(self._h)
        self._h = None

    __del__ = close

    def _use_current_stream(self):
        torch = _torch()
        _check(self._h, _lib.fkk_plan_set_stream(self._h, _vp(torch.cuda.current_stream(self.device).cuda_stream)))

    def _out(self, n_rows: int, out):
        torch = _torch()
        if out is None:
            dt = torch.float32 if self.imag_only else torch.complex64
            out = torch.empty((n_rows, self.n_freq), dtype=dt, device=f"cuda:{self.device}")
        return out

    def _check_cube(self, I, Iref):
        torch = _torch()
        want = torch.float64 if self.in_dtype == "f64" else torch.float32
        if I.dtype != want or Iref.dtype != want:
            raise TypeError(f"cube and reference must be {want}")
        if I.dim() != 2 or I.shape[1] != self.n_freq or Iref.numel() != self.n_freq:
            raise ValueError("cube must be N x M and reference length M")

    def sync(self):
        _check(self._h, _lib.fkk_plan_sync(self._h))

    # -------------------------------------------------------------- calls
    def svd(self, I, Iref):
        torch = _torch()
        self._check_cube(I, Iref)
        self._use_current_stream()
        V = torch.empty((self.rank_k, self.n_freq), dtype=torch.float32, device=I.device)  # = M x k col-major
        s = np.zeros(self.rank_k)
        _check(self._h, _lib.fkk_svd(self._h, _dev_ptr(I, "I"), I.shape[0], _dev_ptr(Iref, "I_ref"), _dev_ptr(V, "V"),
                                     s.ctypes.data_as(_dp)))
        return V, s

    def transform(self, I, Iref, out=None, return_basis: bool = False):
        self._check_cube(I, Iref)
        self._use_current_stream()
        out = self._out(I.shape[0], out)
        bh = _vp()
        _check(self._h, _lib.fkk_transform(self._h, _dev_ptr(I, "I"), I.shape[0], _dev_ptr(Iref, "I_ref"),
                                           _dev_ptr(out, "out"), ctypes.byref(bh) if return_basis else None))
        return (out, Basis(bh)) if return_basis else out

    def transform_from(self, I, Iref, V, s, q, out=None):
        """F5..F11 with given V (k x M fp32 CUDA tensor = M x k column-major), s (k), q (global rows)."""
        self._check_cube(I, Iref)
        self._use_current_stream()
        out = self._out(I.shape[0], out)
        s = np.ascontiguousarray(s, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.int64)
        _check(self._h, _lib.fkk_transform_from(self._h, _dev_ptr(I, "I"), I.shape[0], _dev_ptr(Iref, "I_ref"),
                                                _dev_ptr(V, "V"), s.ctypes.data_as(_dp),
                                                q.ctypes.data_as(ctypes.POINTER(_i64)), len(q), _dev_ptr(out, "out")))
        return out

    def apply(self, basis: Basis, I, out=None):
        self._use_current_stream()
        out = self._out(I.shape[0], out)
        _check(self._h, _lib.fkk_apply_trained_basis(self._h, basis.handle, _dev_ptr(I, "I"), I.shape[0],
                                                     _dev_ptr(out, "out")))
        return out

    def direct(self, I, Iref, out=None):
        self._check_cube(I, Iref)
        self._use_current_stream()
        out = self._out(I.shape[0], out)
        _check(self._h, kk_direct_batch_raw(self._h, I, Iref, out))
        return out

    def conventional(self, I, Iref, k_keep, out=None):
        """fkk_conventional: rank-k_keep SVD denoise of the raw cube, then the direct KK (Fig. 1(a))."""
        self._check_cube(I, Iref)
        self._use_current_stream()
        out = self._out(I.shape[0], out)
        _check(self._h, _lib.fkk_conventional(self._h, _dev_ptr(I, "I"), I.shape[0], _dev_ptr(Iref, "I_ref"),
                                              int(k_keep), _dev_ptr(out, "out")))
        return out

    # host-buffer variants (numpy arrays or pinned CPU torch tensors)
    def _host_ptr(self, a):
        if isinstance(a, np.ndarray):
            if not a.flags.c_contiguous:
                raise ValueError("host arrays must be C-contiguous")
            return _vp(a.ctypes.data)
        return _vp(a.data_ptr())

    def transform_host(self, I, Iref, out, return_basis: bool = False):
        bh = _vp()
        _check(self._h, _lib.fkk_transform_host(self._h, self._host_ptr(I), I.shape[0], self._host_ptr(Iref),
                                                self._host_ptr(out), ctypes.byref(bh) if return_basis else None))
        return Basis(bh) if return_basis else None

    def transform_host_stream(self, cubes, Iref, outs) -> np.ndarray:
        """fkk_transform_host_stream: one transform per host cube (pinned; equal row counts), the copies
        of neighbouring cubes overlapping the transforms; returns the per-cube latencies (ms)."""
        n = len(cubes)
        if len(outs) != n or any(c.shape != cubes[0].shape for c in cubes):
            raise ValueError("cubes / outs: equal counts and shapes")
        ins = (_vp * max(n, 1))(*[self._host_ptr(c) for c in cubes])
        ous = (_vp * max(n, 1))(*[self._host_ptr(o) for o in outs])
        ms = np.zeros(max(n, 1), dtype=np.float32)
        _check(self._h, _lib.fkk_transform_host_stream(self._h, ins, n, cubes[0].shape[0] if n else 1,
                                                       self._host_ptr(Iref), ous,
                                                       ms.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return ms[:n]

    def direct_host(self, I, Iref, out):
        _check(self._h, _lib.kk_direct_batch_host(self._h, self._host_ptr(I), I.shape[0], self._host_ptr(Iref),
                                                  self._host_ptr(out)))

    def apply_stream(self, basis: Basis, I, out, batch: int) -> np.ndarray:
        """fkk_apply_trained_basis_stream: host cube (pinned) -> host output in `batch`-spectrum batches;
        returns the per-batch end-to-end latencies (ms)."""
        nb = max(1, -(-I.shape[0] // batch))
        ms = np.zeros(nb, dtype=np.float32)
        _check(self._h, _lib.fkk_apply_trained_basis_stream(self._h, basis.handle, self._host_ptr(I), I.shape[0], batch,
                                                            self._host_ptr(out),
                                                            ms.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
        return ms

    def apply_host(self, basis: Basis, I, out):
        _check(self._h, _lib.fkk_apply_trained_basis_host(self._h, basis.handle, self._host_ptr(I), I.shape[0],
                                                          self._host_ptr(out)))

    # -------------------------------------------------------------- diagnostics
    def stage(self, name: str) -> np.ndarray:
        sid = STAGES[name]
        nbytes = _lib.fkk_stage_size(self._h, sid)
        dtype = {"US": np.float32, "B": np.float32, "Q": np.int64}.get(name, np.float64)
        buf = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
        _check(self._h, _lib.fkk_get_stage(self._h, sid, _vp(buf.ctypes.data), nbytes, 0))
        M, k = self.n_freq, self.rank_k
        if name == "G":
            return buf.reshape(M, M)
        if name == "V":
            return buf.reshape(k, M).T          # M x k
        if name == "US":
            return buf.reshape(-1, k)
        if name in ("HV", "PHI_PEC", "V_SEC"):
            return buf.reshape(k, M)
        if name == "PHI_ERR":
            return buf.reshape(-1, M)
        if name == "B":
            return buf.reshape(k, M, 2)
        return buf

    def stage_times(self) -> dict:
        cap = 64
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        n = _lib.fkk_stage_times(self._h, names, ms, cap)
        out: dict = {}
        for i in range(n):
            key = names[i].decode()
            out[key] = out.get(key, 0.0) + float(ms[i])
        return out

    @property
    def launches(self) -> int:
        return int(_lib.fkk_last_launch_count(self._h))

    def als_solves(self) -> int:
        """ALS solves summed over the direct-path spectra since the last query (then reset)."""
        return int(_lib.fkk_debug_als_solves(self._h))


def kk_direct_batch_raw(handle, I, Iref, out) -> int:
    return _lib.kk_direct_batch(handle, _dev_ptr(I, "I"), I.shape[0], _dev_ptr(Iref, "I_ref"), _dev_ptr(out, "out"))


# ------------------------------------------------------------------ C-ABI-named functions
def fkk_plan_create(n_freq, rank_k, max_rows, **kw) -> Plan:
    return Plan(n_freq, rank_k, max_rows, **kw)


def fkk_svd(plan: Plan, I, Iref):
    return plan.svd(I, Iref)


def fkk_transform(plan: Plan, I, Iref, out=None, return_basis=False):
    return plan.transform(I, Iref, out, return_basis)


def fkk_transform_from(plan: Plan, I, Iref, V, s, q, out=None):
    return plan.transform_from(I, Iref, V, s, q, out)


def fkk_apply_trained_basis(plan: Plan, basis: Basis, I, out=None):
    return plan.apply(basis, I, out)


def kk_direct_batch(plan: Plan, I, Iref, out=None):
    return plan.direct(I, Iref, out)


def fkk_debug_tc_mma(mode: int, A, B):
    """Tensor-core self-test: D = tf32(A) tf32(B)^T through one tcgen05.mma (A 128x8, B Nx8 CUDA fp32)."""
    torch = _torch()
    D = torch.zeros((128, B.shape[0]), dtype=torch.float32, device=A.device)
    _check(None, _lib.fkk_debug_tc_mma(mode, _dev_ptr(A, "A"), _dev_ptr(B, "B"), _dev_ptr(D, "D"), B.shape[0]))
    return D


def fkk_debug_eig_topk(G, k: int):
    """The GPU eigensolver (F4) on a symmetric CUDA fp64 matrix G: returns (V: M x k, lam: k), CUDA."""
    torch = _torch()
    M = G.shape[0]
    V = torch.zeros((k, M), dtype=torch.float64, device=G.device)
    lam = torch.zeros(k, dtype=torch.float64, device=G.device)
    _check(None, _lib.fkk_debug_eig_topk(_dev_ptr(G, "G"), M, k, _dev_ptr(V, "V"), _dev_ptr(lam, "lam")))
    return V.T, lam


def fkk_debug_tridiag(G):
    """The tridiagonalisation alone: returns (d, e, tau) as CUDA fp64 tensors."""
    torch = _torch()
    M = G.shape[0]
    out = torch.zeros(3 * M, dtype=torch.float64, device=G.device)
    _check(None, _lib.fkk_debug_tridiag(_dev_ptr(G, "G"), M, _dev_ptr(out, "out")))
    return out[:M], out[M:2 * M], out[2 * M:]


def fkk_debug_eig_path(M: int) -> int:
    return int(_lib.fkk_debug_eig_path(M))


def fkk_range_finder_omega(seed: int, M: int, l: int) -> np.ndarray:
    """The range finder's Gaussian test matrix Omega (M x l), generated by the library (host code)."""
    out = np.zeros((M, l))
    if _lib.fkk_range_finder_omega(seed, M, l, out.ctypes.data_as(_dp)) != 0:
        raise FkkError(1, "bad arguments")
    return out


_ALLGATHER = ctypes.CFUNCTYPE(_i32, _vp, _vp, _vp, ctypes.c_size_t)
_ALLRED_F64 = ctypes.CFUNCTYPE(_i32, _vp, _dp, ctypes.c_size_t)
_ALLRED_I32 = ctypes.CFUNCTYPE(_i32, _vp, ctypes.POINTER(_i32), ctypes.c_size_t)


class HostCollectives(ctypes.Structure):
    _fields_ = [("ctx", _vp), ("world_size", _i32), ("rank", _i32), ("allgather", _ALLGATHER),
                ("allreduce_sum_f64", _ALLRED_F64), ("allreduce_max_i32", _ALLRED_I32)]


def fkk_exchange_selftest(world: int, rank: int, allgather, allreduce_sum, allreduce_max, n_rows: int, M: int, k: int,
                          shards: int, G: np.ndarray, ext_val: np.ndarray, ext_idx: np.ndarray, US_local: np.ndarray,
                          flags: int):
    """Run the sharded transform's exchange sequence (the library's C++ code) on host data through the
    given collectives (python callables on numpy arrays: allgather(send_bytes) -> world x bytes,
    allreduce_sum(float64 array) in place, allreduce_max(int32 array) in place)."""
    def ag(ctx, send, recv, nbytes):
        try:
            src = np.ctypeslib.as_array(ctypes.cast(send, ctypes.POINTER(ctypes.c_uint8)), (nbytes,)).copy()
            out = allgather(src)
            ctypes.memmove(recv, out.ctypes.data, out.nbytes)
            return 0
        except Exception:
            return 1

    def ars(ctx, data, n):
        try:
            a = np.ctypeslib.as_array(data, (n,))
            a[:] = allreduce_sum(a.copy())
            return 0
        except Exception:
            return 1

    def arm(ctx, data, n):
        try:
            a = np.ctypeslib.as_array(data, (n,))
            a[:] = allreduce_max(a.copy())
            return 0
        except Exception:
            return 1

    cb = (_ALLGATHER(ag), _ALLRED_F64(ars), _ALLRED_I32(arm))
    hc = HostCollectives(None, world, rank, *cb)
    G = np.ascontiguousarray(G, dtype=np.float64)
    ev = np.ascontiguousarray(ext_val, dtype=np.float32)
    ei = np.ascontiguousarray(ext_idx, dtype=np.int64)
    us = np.ascontiguousarray(US_local, dtype=np.float32)
    fl = _i32(flags)
    row0, ng, nq = _i64(), _i64(), _i32()
    q = np.zeros(2 * k, dtype=np.int64)
    X = np.zeros((2 * k, k))
    st = _lib.fkk_exchange_selftest(ctypes.byref(hc), n_rows, M, k, shards, G.ctypes.data_as(_dp),
                                    ev.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                    ei.ctypes.data_as(ctypes.POINTER(_i64)),
                                    us.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), ctypes.byref(fl),
                                    ctypes.byref(row0), ctypes.byref(ng), q.ctypes.data_as(ctypes.POINTER(_i64)),
                                    ctypes.byref(nq), X.ctypes.data_as(_dp))
    if st != FKK_OK:
        raise FkkError(st, "exchange self-test failed")
    return dict(row0=row0.value, n_global=ng.value, G=G, q=q[:nq.value], X=X[:nq.value], flags=fl.value)


def fkk_get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(None, _lib.fkk_get_nccl_unique_id(buf))
    return buf.raw


def fkk_host_eig_topk(G: np.ndarray, k: int):
    G = np.ascontiguousarray(G, dtype=np.float64)
    M = G.shape[0]
    V = np.zeros((k, M))
    lam = np.zeros(k)
    st = _lib.fkk_host_eig_topk(G.ctypes.data_as(_dp), M, k, V.ctypes.data_as(_dp), lam.ctypes.data_as(_dp))
    if st != FKK_OK:
        raise FkkError(st, "host eigensolver failed")
    return V.T.copy(), lam


def fkk_shard_range(n_global: int, world: int, rank: int):
    a, b = _i64(), _i64()
    _lib.fkk_shard_range(n_global, world, rank, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def fkk_merge_extremes(vals: np.ndarray, idx: np.ndarray, k: int) -> np.ndarray:
    """vals/idx: world x k x 2 (0 = max, 1 = min); returns sorted unique q."""
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    world = vals.shape[0]
    out = np.zeros(2 * k, dtype=np.int64)
    n = _lib.fkk_merge_extremes(vals.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                idx.ctypes.data_as(ctypes.POINTER(_i64)), world, k,
                                out.ctypes.data_as(ctypes.POINTER(_i64)))
    return out[:n]
