"""Python binding of the B200 DME hot path (libdme.so, C ABI in include/dme.h).

Argument marshalling only: every step of the method runs in the CUDA library. PyTorch provides
the device workspace, the stream and (for world_size > 1) the process group used to broadcast
the NCCL unique id. There is NO CPU fallback: importing this package on a machine where the
extension is missing raises, and creating a Solver without a CUDA device raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DME_LIB: another in-tree build of the same library (A/B measurements in tools/); no fallback
LIB_PATH = os.environ.get("DME_LIB") or os.path.join(_HERE, "libdme.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

SCHEMES = {"lie": 0, "strang": 1}
COMPOSITIONS = {"F1F2": 0, "F12": 1, "F12F3": 2, "F1F2F3": 3, "F1F3F2": 4, "F12F4": 5,
                "F1F2F4": 6, "F1F4F2": 7, "F12F3F4": 8, "F1F2F3F4": 9}
FLOWS = {"T1": 0, "T2": 1, "T3": 2, "T4": 3, "T4_euler": 4, "T12": 5, "compress": 6}
STATUS = {0: "ok", 1: "invalid argument", 2: "dimension error", 3: "configuration error",
          4: "singular system", 5: "numerical failure", 6: "capacity exceeded", 7: "CUDA error",
          8: "NCCL error", 9: "out of memory", 10: "context poisoned"}

_dp = ctypes.POINTER(ctypes.c_double)


class _Problem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("A", _dp), ("p", ctypes.c_int64), ("C", _dp),
                ("m", ctypes.c_int64), ("B", _dp), ("R", _dp), ("S", _dp),
                ("r0", ctypes.c_int64), ("L0", _dp), ("D0", _dp), ("M", _dp),
                ("A_nnz", ctypes.c_int64), ("A_rowptr", ctypes.POINTER(ctypes.c_int64)),
                ("A_colind", ctypes.POINTER(ctypes.c_int32)), ("A_values", _dp),
                ("S_nnz", ctypes.c_int64), ("S_rowptr", ctypes.POINTER(ctypes.c_int64)),
                ("S_colind", ctypes.POINTER(ctypes.c_int32)), ("S_values", _dp)]


class _Options(ctypes.Structure):
    _fields_ = [("h", ctypes.c_double), ("trunc_tol", ctypes.c_double),
                ("rank_cap", ctypes.c_int32), ("quad_nodes", ctypes.c_int32),
                ("quad_subpanels", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("world_size", ctypes.c_int32),
                ("world_rank", ctypes.c_int32), ("nccl_uid", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("big_inputs_on_device", ctypes.c_int32), ("no_fsal", ctypes.c_int32),
                ("e_pass", ctypes.c_int32), ("expm", ctypes.c_int32),
                ("compression", ctypes.c_int32), ("virtual_world", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("steps", ctypes.c_int64), ("rank", ctypes.c_int64),
                ("max_rank", ctypes.c_int64), ("q_half", ctypes.c_int64),
                ("q_full", ctypes.c_int64), ("squarings", ctypes.c_int32),
                ("quad_panels", ctypes.c_int32), ("panel_width", ctypes.c_double),
                ("pade_min_pivot", ctypes.c_double), ("last_drop", ctypes.c_double),
                ("e_passes", ctypes.c_int64), ("compressions", ctypes.c_int64),
                ("init_seconds", ctypes.c_double), ("kernel_launches", ctypes.c_int64),
                ("prof_passes", ctypes.c_int64), ("prof_epass_seconds", ctypes.c_double),
                ("prof_epass_flops", ctypes.c_double), ("prof_epass_bytes", ctypes.c_double),
                ("prof_gram_seconds", ctypes.c_double), ("prof_small_seconds", ctypes.c_double),
                ("prof_apply_seconds", ctypes.c_double), ("eig_fallbacks", ctypes.c_int64),
                ("ozaki_passes", ctypes.c_int64), ("cheb_degree", ctypes.c_int64),
                ("expm_chebyshev", ctypes.c_int64)]


_ctx_p = ctypes.c_void_p
_lib.dme_default_options.argtypes = [ctypes.POINTER(_Options)]
_lib.dme_status_string.restype = ctypes.c_char_p
_lib.dme_last_error.restype = ctypes.c_char_p
for _name, _args in {
    "dme_workspace_size": [ctypes.POINTER(_Problem), ctypes.POINTER(_Options),
                           ctypes.POINTER(ctypes.c_size_t)],
    "dme_get_unique_id": [ctypes.c_void_p],
    "dme_shard_rows": [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
    "dme_dle_init": [ctypes.POINTER(_Problem), ctypes.POINTER(_Options), ctypes.POINTER(_ctx_p)],
    "dme_dre_init": [ctypes.POINTER(_Problem), ctypes.POINTER(_Options), ctypes.POINTER(_ctx_p)],
    "dme_split_step": [_ctx_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64],
    "dme_get_factor": [_ctx_p, ctypes.POINTER(ctypes.c_int64), _dp, _dp, ctypes.c_int64],
    "dme_extrapolate": [_ctx_p, _ctx_p, ctypes.POINTER(ctypes.c_int64), _dp, _dp, ctypes.c_int64],
    "dme_get_stats": [_ctx_p, ctypes.POINTER(_Stats)],
    "dme_set_profiling": [_ctx_p, ctypes.c_int32],
    "dme_destroy": [_ctx_p],
    "dme_debug_apply": [_ctx_p, ctypes.c_int32, ctypes.c_double],
    "dme_debug_set_factor": [_ctx_p, ctypes.c_int64, _dp],
    "dme_debug_get_exp": [_ctx_p, ctypes.c_int32, _dp],
    "dme_debug_set_exp": [_ctx_p, ctypes.c_int32, _dp],
    "dme_debug_get_integral": [_ctx_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), _dp,
                               ctypes.c_int64],
    "dme_debug_matmul": [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _dp, _dp, _dp],
    "dme_debug_matmul_ozaki": [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _dp, _dp, _dp],
    "dme_debug_complement": [ctypes.c_int64, ctypes.c_int64, _dp, _dp],
    "dme_debug_small_stats": [_ctx_p, _dp],
    "dme_cheb_coeffs": [ctypes.c_double, ctypes.c_double, _dp, ctypes.c_int64,
                        ctypes.POINTER(ctypes.c_int32)],
}.items():
    if os.environ.get("DME_LIB") and not hasattr(_lib, _name):
        continue  # an older build under A/B measurement may lack newer test hooks
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = ctypes.c_int

EXPORTED = ["dme_default_options", "dme_status_string", "dme_last_error", "dme_workspace_size",
            "dme_get_unique_id", "dme_shard_rows", "dme_dle_init", "dme_dre_init", "dme_split_step",
            "dme_get_factor", "dme_extrapolate", "dme_get_stats", "dme_set_profiling", "dme_destroy", "dme_debug_apply",
            "dme_debug_set_factor", "dme_debug_get_exp", "dme_debug_set_exp", "dme_debug_get_integral",
            "dme_debug_small_stats", "dme_debug_matmul", "dme_debug_matmul_ozaki", "dme_cheb_coeffs",
            "dme_debug_complement"]


class DmeError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        msg = _lib.dme_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(code, code)} ({msg})")


def _check(code, where):
    if code != 0:
        raise DmeError(code, where)


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Options:
    h: float
    trunc_tol: float = 1e-16
    rank_cap: int = 0
    quad_nodes: int = 14
    quad_subpanels: int = 1


def shard_rows(n: int, world: int, rank: int):
    """(row0, rows, nloc) of the E row shard owned by `rank` (host logic of the C library)."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.dme_shard_rows(n, world, rank, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
           "dme_shard_rows")
    return a.value, b.value, c.value


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.dme_get_unique_id(buf), "dme_get_unique_id")
    return buf.raw


E_PASS = {"auto": 0, "dmma": 1}
EXPM = {"auto": 0, "pade": 1}
COMPRESSION = {"refined": 0, "gram": 1}


def cheb_coeffs(gamma: float, tol: float = 2.0 ** -56) -> np.ndarray:
    """Host routine of the sparse-A path: e^{-gamma} I_k(gamma), k = 0..K, K the degree whose
    coefficient tail 2 sum_{j>K} is <= tol (dme_cheb_coeffs; no device needed)."""
    out = np.zeros(4096)
    K = ctypes.c_int32(0)
    _check(_lib.dme_cheb_coeffs(gamma, tol, _ptr(out), out.size, ctypes.byref(K)), "dme_cheb_coeffs")
    return out[:K.value + 1].copy()


def _is_sparse(A) -> bool:
    return hasattr(A, "tocsr") and hasattr(A, "nnz")


class Solver:
    """One problem on one GPU (or one rank of a row-sharded multi-GPU run)."""

    def __init__(self, A, C=None, L0=None, D0=None, B=None, R=None, S=None, M=None, *, h,
                 trunc_tol=1e-16,
                 rank_cap=0, quad_nodes=14, quad_subpanels=1, device=None, stream=None,
                 world_size=1, world_rank=0, nccl_uid: Optional[bytes] = None, fsal=True,
                 e_pass="auto", expm="auto", compression="refined", virtual_world=0, poison_workspace=False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1805_08990_b200.Solver needs a CUDA device (no CPU fallback)")
        self._torch = torch
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        # A and S may be CUDA tensors (float64, contiguous): then they are read device-to-device
        on_dev = isinstance(A, torch.Tensor) and A.is_cuda
        sparse = _is_sparse(A)
        self._csrS = None
        if _is_sparse(S):  # CSR S (T4 by sparse x skinny products); host arrays
            cs = S.tocsr()
            self._csrS = (np.ascontiguousarray(cs.indptr, dtype=np.int64),
                          np.ascontiguousarray(cs.indices, dtype=np.int32),
                          np.ascontiguousarray(cs.data, dtype=np.float64))
            S = None
        if sparse:  # CSR host arrays; the library builds its device layout from them
            csr = A.tocsr()
            self._csr = (np.ascontiguousarray(csr.indptr, dtype=np.int64),
                         np.ascontiguousarray(csr.indices, dtype=np.int32),
                         np.ascontiguousarray(csr.data, dtype=np.float64))
            self._keep = [None, _f64(C), _f64(B), _f64(R), _f64(S), _f64(L0), _f64(D0), _f64(M)]
            A_, C_, B_, R_, S_, L0_, D0_, M_ = self._keep
            pA, pS, pM = None, _ptr(S_), _ptr(M_)
        elif on_dev:
            if A.dtype != torch.float64 or not A.is_contiguous():
                raise ValueError("device A must be a contiguous float64 CUDA tensor")
            if S is not None and not (isinstance(S, torch.Tensor) and S.is_cuda and
                                      S.dtype == torch.float64 and S.is_contiguous()):
                raise ValueError("with a device A, S must be a contiguous float64 CUDA tensor")
            if M is not None and not (isinstance(M, torch.Tensor) and M.is_cuda and
                                      M.dtype == torch.float64 and M.is_contiguous()):
                raise ValueError("with a device A, M must be a contiguous float64 CUDA tensor")
            dptr = lambda t: None if t is None else ctypes.cast(t.data_ptr(), _dp)
            self._keep = [A, _f64(C), _f64(B), _f64(R), S, _f64(L0), _f64(D0), M]
            A_, C_, B_, R_, S_, L0_, D0_, M_ = self._keep
            pA, pS, pM = dptr(A_), dptr(S_), dptr(M_)
        else:
            self._keep = [_f64(A), _f64(C), _f64(B), _f64(R), _f64(S), _f64(L0), _f64(D0), _f64(M)]
            A_, C_, B_, R_, S_, L0_, D0_, M_ = self._keep
            pA, pS, pM = _ptr(A_), _ptr(S_), _ptr(M_)
        n = A.shape[0]
        self.n = n
        pr = _Problem(n=n, A=pA, p=0 if C_ is None else C_.shape[0], C=_ptr(C_),
                      m=0 if B_ is None else B_.shape[1], B=_ptr(B_), R=_ptr(R_), S=pS,
                      r0=0 if L0_ is None else L0_.shape[1], L0=_ptr(L0_), D0=_ptr(D0_), M=pM)
        if self._csrS is not None:
            rp, ci, vv = self._csrS
            pr.S_nnz = vv.size
            pr.S_rowptr = rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            pr.S_colind = ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            pr.S_values = _ptr(vv)
        if sparse:
            rp, ci, vv = self._csr
            pr.A_nnz = vv.size
            pr.A_rowptr = rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            pr.A_colind = ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            pr.A_values = _ptr(vv)
        self._pr = pr
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
        self._uid = uid
        opt = _Options(h=h, trunc_tol=trunc_tol, rank_cap=rank_cap, quad_nodes=quad_nodes,
                       quad_subpanels=quad_subpanels, device=dev.index,
                       stream=self.stream.cuda_stream, world_size=world_size,
                       world_rank=world_rank, nccl_uid=ctypes.cast(uid, ctypes.c_void_p) if uid else None,
                       workspace=None, workspace_bytes=0, big_inputs_on_device=1 if on_dev else 0,
                       no_fsal=0 if fsal else 1, e_pass=E_PASS[e_pass], expm=EXPM[expm],
                       compression=COMPRESSION[compression], virtual_world=virtual_world)
        nbytes = ctypes.c_size_t(0)
        _check(_lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(opt), ctypes.byref(nbytes)),
               "dme_workspace_size")
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=dev)
        if poison_workspace:  # test hook: the library must not rely on zeroed caller memory
            self.workspace.fill_(0xFF)
        opt.workspace = self.workspace.data_ptr()
        opt.workspace_bytes = self.workspace.numel()
        self._opt = opt
        self._ctx = _ctx_p()
        init = _lib.dme_dre_init if pr.m > 0 else _lib.dme_dle_init
        with torch.cuda.device(dev):
            _check(init(ctypes.byref(pr), ctypes.byref(opt), ctypes.byref(self._ctx)), "dme_init")
        self.h = h

    # ---------------------------------------------------------------- stepping
    def split_step(self, scheme: str, composition: str, nsteps: int = 1):
        _check(_lib.dme_split_step(self._ctx, SCHEMES[scheme], COMPOSITIONS[composition], nsteps),
               "dme_split_step")

    def get_factor(self):
        r = ctypes.c_int64(0)
        _check(_lib.dme_get_factor(self._ctx, ctypes.byref(r), None, None, 0), "dme_get_factor")
        L = np.zeros((self.n, r.value))
        D = np.zeros((r.value, r.value))
        _check(_lib.dme_get_factor(self._ctx, ctypes.byref(r), _ptr(L), _ptr(D), r.value),
               "dme_get_factor")
        return L, D

    def stats(self) -> dict:
        s = _Stats()
        _check(_lib.dme_get_stats(self._ctx, ctypes.byref(s)), "dme_get_stats")
        return {f: getattr(s, f) for f, _ in _Stats._fields_}

    def set_profiling(self, on: bool):
        _check(_lib.dme_set_profiling(self._ctx, 1 if on else 0), "dme_set_profiling")

    # ---------------------------------------------------------------- test hooks
    def debug_apply(self, flow: str, tau: float):
        _check(_lib.dme_debug_apply(self._ctx, FLOWS[flow], tau), "dme_debug_apply")

    def debug_set_factor(self, L):
        L = _f64(L)
        _check(_lib.dme_debug_set_factor(self._ctx, L.shape[1], _ptr(L)), "dme_debug_set_factor")

    def debug_get_exp(self, which: int):
        E = np.zeros((self.n, self.n))
        _check(_lib.dme_debug_get_exp(self._ctx, which, _ptr(E)), "dme_debug_get_exp")
        return E

    def debug_set_exp(self, which: int, E):
        E = _f64(E)
        _check(_lib.dme_debug_set_exp(self._ctx, which, _ptr(E)), "dme_debug_set_exp")

    def debug_get_integral(self, which: int):
        q = ctypes.c_int64(0)
        _check(_lib.dme_debug_get_integral(self._ctx, which, ctypes.byref(q), None, 0), "integral")
        L = np.zeros((self.n, q.value))
        _check(_lib.dme_debug_get_integral(self._ctx, which, ctypes.byref(q), _ptr(L), q.value),
               "integral")
        return L

    def debug_small_stats(self):
        out = np.zeros(16)
        _check(_lib.dme_debug_small_stats(self._ctx, _ptr(out)), "dme_debug_small_stats")
        return out

    def close(self):
        if getattr(self, "_ctx", None):
            _lib.dme_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def extrapolate(fine: "Solver", coarse: "Solver"):
    """Richardson-extrapolated Strang: (4 P_fine - P_coarse)/3 as (L, D), D diagonal and possibly
    indefinite (dme_extrapolate; fine: step h/2 after 2N steps, coarse: step h after N steps)."""
    r = ctypes.c_int64(0)
    _check(_lib.dme_extrapolate(fine._ctx, coarse._ctx, ctypes.byref(r), None, None, 0),
           "dme_extrapolate")
    L = np.zeros((fine.n, r.value))
    D = np.zeros((r.value, r.value))
    _check(_lib.dme_extrapolate(fine._ctx, coarse._ctx, ctypes.byref(r), _ptr(L), _ptr(D), r.value),
           "dme_extrapolate")
    return L, D


def matmul_ozaki(A, B):
    """C = A @ B through the int8 digit-slicing (Ozaki) kernel of the E pass (B.shape[1] <= 64)."""
    A, B = _f64(A), _f64(B)
    C = np.zeros((A.shape[0], B.shape[1]))
    _check(_lib.dme_debug_matmul_ozaki(A.shape[0], B.shape[1], A.shape[1], _ptr(A), _ptr(B),
                                       _ptr(C)), "dme_debug_matmul_ozaki")
    return C


def complement_basis(W):
    """Orthonormal basis (k x (k - kb)) of the complement of span(W) (W: k x kb, orthonormal
    columns) through the refined compression's complement-basis kernel (test hook)."""
    W = _f64(W)
    k, kb = W.shape
    U = np.zeros((k, k - kb))
    _check(_lib.dme_debug_complement(k, kb, _ptr(W), _ptr(U)), "dme_debug_complement")
    return U


def matmul(A, B):
    """C = A @ B through the library's FP64 DMMA GEMM (host arrays in and out; test hook)."""
    A, B = _f64(A), _f64(B)
    C = np.zeros((A.shape[0], B.shape[1]))
    _check(_lib.dme_debug_matmul(A.shape[0], B.shape[1], A.shape[1], _ptr(A), _ptr(B), _ptr(C)),
           "dme_debug_matmul")
    return C


def problem_kwargs(prob) -> dict:
    """workloads.Problem -> Solver keyword arguments (data only)."""
    return dict(A=prob.A, C=prob.C, L0=prob.L0 if prob.L0 is not None and prob.L0.shape[1] else None,
                D0=prob.D0 if prob.L0 is not None and prob.L0.shape[1] else None, B=prob.B,
                R=prob.R, S=prob.S, M=getattr(prob, "M", None))
