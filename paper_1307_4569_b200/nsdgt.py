"""Thin ctypes binding of the C ABI in ``include/nsdgt.h`` (argument marshalling only).

Every step of the transform runs in ``libnsdgt.so`` (hand-written sm_100a kernels;
cuFFT only for the length-L FFTs of the frequency-shear branch).  There is no CPU
fallback: if the library is missing this module raises at import.  PyTorch is used
only for device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnsdgt.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1307_4569_b200.build` "
                      "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

DGT_OK, DGT_EINVAL, DGT_EILLEGAL_LENGTH, DGT_ECUDA, DGT_ECUFFT, DGT_ENOMEM, DGT_EUNSUPPORTED = 0, 2, 4, 5, 6, 7, 8
DGT_C64, DGT_C128 = 1, 2
DGT_REAL_INPUT, DGT_G_ON_HOST, DGT_SHEAR_PAPER, DGT_FORCE_GENERIC = 1, 2, 4, 8
BRANCH_NAMES = {0: "separable", 1: "time", 2: "freq"}

_FIELDS = ["L", "a", "M", "lambda1", "lambda2", "b", "N", "s", "L_min", "branch", "s0", "s1", "b_r", "a_r",
           "M_r", "N_r", "ia", "iM", "iN", "ib", "c", "d", "p", "q", "C1", "C2", "C3", "C4", "C5", "C6",
           "chirp_sigma", "pre_sigma", "chunk", "workspace_bytes", "kernel_path"]


class LatticeInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in _FIELDS]

    def to_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f in _FIELDS}


class KernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("ms", ctypes.c_double),
                ("bytes", ctypes.c_double), ("flops", ctypes.c_double)]


EXPORTS = ["dgt_lattice_plan", "dgt_plan", "dgt_plan_fir", "dgt_plan_multiwindow", "dgt_execute", "dgt_execute_inverse", "dgt_window_dual", "dgt_execute_host",
           "dgt_destroy",
           "dgt_plan_query",
           "dgt_launches_per_execute", "dgt_profile_begin", "dgt_profile_end", "dgt_strerror", "dgt_last_error",
           "dgt_last_lmin", "dgt_version"]

_I64, _P, _INT = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
_lib.dgt_lattice_plan.argtypes = [_I64] * 5 + [_INT, _INT, _I64, _I64, ctypes.POINTER(LatticeInfo)]
_lib.dgt_lattice_plan.restype = _INT
_lib.dgt_plan.argtypes = [ctypes.POINTER(_P)] + [_I64] * 5 + [_P, _INT, _INT, _I64, _INT, _I64, _I64, _P]
_lib.dgt_plan.restype = _INT
_lib.dgt_plan_fir.argtypes = [ctypes.POINTER(_P)] + [_I64] * 5 + [_P, _I64, _I64, _INT, _INT, _P]
_lib.dgt_plan_fir.restype = _INT
_lib.dgt_plan_multiwindow.argtypes = [ctypes.POINTER(_P)] + [_I64] * 5 + [_P, _INT, _INT, _P]
_lib.dgt_plan_multiwindow.restype = _INT
_lib.dgt_execute.argtypes = [_P, _P, _P, _I64, _P]
_lib.dgt_execute.restype = _INT
_lib.dgt_execute_inverse.argtypes = [_P, _P, _P, _I64, _P]
_lib.dgt_execute_inverse.restype = _INT
_lib.dgt_window_dual.argtypes = [_P, _INT, _P, _INT, _P]
_lib.dgt_window_dual.restype = _INT
_lib.dgt_execute_host.argtypes = [_P, _P, _P, _I64, _P]
_lib.dgt_execute_host.restype = _INT
_lib.dgt_destroy.argtypes = [_P]
_lib.dgt_destroy.restype = _INT
_lib.dgt_plan_query.argtypes = [_P, ctypes.POINTER(LatticeInfo)]
_lib.dgt_plan_query.restype = _INT
_lib.dgt_launches_per_execute.argtypes = [_P, _I64]
_lib.dgt_launches_per_execute.restype = _I64
_lib.dgt_profile_begin.argtypes = [_P]
_lib.dgt_profile_begin.restype = _INT
_lib.dgt_profile_end.argtypes = [_P, ctypes.POINTER(KernelStat), _INT, ctypes.POINTER(_INT)]
_lib.dgt_profile_end.restype = _INT
_lib.dgt_strerror.argtypes = [_INT]
_lib.dgt_strerror.restype = ctypes.c_char_p
_lib.dgt_last_error.restype = ctypes.c_char_p
_lib.dgt_last_lmin.restype = _I64
_lib.dgt_version.restype = ctypes.c_char_p


class DgtError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.dgt_last_error().decode(errors="replace")
        msg = f"{where}: {_lib.dgt_strerror(status).decode()} ({status})"
        if detail:
            msg += f": {detail}"
        if status == DGT_EILLEGAL_LENGTH:
            self.L_min = int(_lib.dgt_last_lmin())
            msg += f" [L_min={self.L_min}]"
        super().__init__(msg)


def _check(status: int, where: str):
    if status != DGT_OK:
        raise DgtError(status, where)


def version() -> str:
    return _lib.dgt_version().decode()


def lattice_plan(L, a, M, lam1, lam2, paper_shear=False, shear=None) -> dict:
    """Host-only planner record (no GPU needed).  ``shear=(s0, s1)`` forces a shear."""
    info = LatticeInfo()
    flags = DGT_SHEAR_PAPER if paper_shear else 0
    s0, s1 = shear if shear is not None else (0, 0)
    _check(_lib.dgt_lattice_plan(L, a, M, lam1, lam2, flags, 1 if shear is not None else 0, s0, s1,
                                 ctypes.byref(info)), "dgt_lattice_plan")
    return info.to_dict()


def _dtype_code(dtype: str) -> int:
    if dtype in ("c64", "complex64", "fp32", "float32"):
        return DGT_C64
    if dtype in ("c128", "complex128", "fp64", "float64"):
        return DGT_C128
    raise ValueError(f"bad dtype {dtype!r}")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """A DGT plan for (L, a, M, lambda1/lambda2) with window ``g`` (length L).

    ``g`` may be a numpy array / CPU tensor (copied from host) or a CUDA tensor.
    ``dtype`` is "c64" or "c128" (working and output precision).
    """

    def __init__(self, L, a, M, lam1, lam2, g, dtype="c64", real_input=False, max_chunk=0, shear=None,
                 paper_shear=False, force_generic=False, stream=None, fir=False, Lb=0, algorithm="shear"):
        """``fir=True``: ``g`` is an FIR window of len(g) <= L taps in FIR order (entries
        [0, ceil(Lg/2)) are times 0.., the rest negative times) and the plan is a shear-OLA plan
        (dgt_plan_fir) with block length ``Lb`` (0 = automatic).  ``algorithm="multiwindow"``:
        the multiwindow comparison algorithm (dgt_plan_multiwindow) instead of the shear
        algorithm."""
        if algorithm not in ("shear", "multiwindow"):
            raise ValueError(f"bad algorithm {algorithm!r}")
        import torch
        code = _dtype_code(dtype)
        # canonical name: every numpy / torch dtype below derives from the code, never from the
        # alias the caller passed ("complex64", "fp32", ...)
        self.dtype = "c64" if code == DGT_C64 else "c128"
        self._np_c = np.complex64 if code == DGT_C64 else np.complex128
        self._cdt = torch.complex64 if code == DGT_C64 else torch.complex128
        self._rdt = torch.float32 if code == DGT_C64 else torch.float64
        self.real_input = bool(real_input)
        flags = (DGT_REAL_INPUT if real_input else 0) | (DGT_SHEAR_PAPER if paper_shear else 0) | \
            (DGT_FORCE_GENERIC if force_generic else 0)
        if isinstance(g, torch.Tensor) and g.is_cuda:
            g_t = g.to(self._cdt).contiguous()
            gptr = g_t.data_ptr()
        else:
            g_np = np.ascontiguousarray(np.asarray(g.cpu() if isinstance(g, torch.Tensor) else g),
                                        dtype=np.complex64 if code == DGT_C64 else np.complex128)
            g_t = g_np
            gptr = g_np.ctypes.data
            flags |= DGT_G_ON_HOST
        ng = int(g_t.numel()) if isinstance(g_t, torch.Tensor) else int(g_t.size)
        if (fir and not 0 < ng <= L) or (not fir and ng != L):
            raise ValueError(f"window has {ng} samples; the plan needs {'1..L' if fir else 'L'} = {L}")
        self._device = torch.cuda.current_device() if torch.cuda.is_available() else -1
        s0, s1 = shear if shear is not None else (0, 0)
        h = ctypes.c_void_p()
        if algorithm == "multiwindow":
            if fir or shear is not None or paper_shear:
                raise ValueError("the multiwindow algorithm takes no FIR window or shear")
            _check(_lib.dgt_plan_multiwindow(ctypes.byref(h), L, a, M, lam1, lam2, ctypes.c_void_p(gptr), code,
                                             flags & ~DGT_SHEAR_PAPER, _stream_ptr(stream)), "dgt_plan_multiwindow")
        elif fir:
            Lg = ng
            _check(_lib.dgt_plan_fir(ctypes.byref(h), L, a, M, lam1, lam2, ctypes.c_void_p(gptr), Lg, int(Lb), code,
                                     flags, _stream_ptr(stream)), "dgt_plan_fir")
        else:
            _check(_lib.dgt_plan(ctypes.byref(h), L, a, M, lam1, lam2, ctypes.c_void_p(gptr), code, flags, max_chunk,
                                 1 if shear is not None else 0, s0, s1, _stream_ptr(stream)), "dgt_plan")
        self._h = h
        del g_t
        info = LatticeInfo()
        _check(_lib.dgt_plan_query(self._h, ctypes.byref(info)), "dgt_plan_query")
        self.info = info.to_dict()
        self.L, self.a, self.M = L, a, M
        self.N = L // a

    def __del__(self):
        self.close()

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.dgt_destroy(h)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self._h = None

    def launches(self, W: int) -> int:
        return int(_lib.dgt_launches_per_execute(self._h, W))

    def profile_begin(self):
        """Record CUDA events around every kernel launch of subsequent executes."""
        _check(_lib.dgt_profile_begin(self._h), "dgt_profile_begin")

    def profile_end(self) -> list:
        """Synchronise the recorded events; per kernel kind: launches, ms, algorithmic bytes, flops."""
        stats = (KernelStat * 16)()
        n = ctypes.c_int(0)
        _check(_lib.dgt_profile_end(self._h, stats, 16, ctypes.byref(n)), "dgt_profile_end")
        return [{"name": stats[i].name.decode(), "launches": int(stats[i].launches), "ms": float(stats[i].ms),
                 "bytes": float(stats[i].bytes), "flops": float(stats[i].flops)} for i in range(min(n.value, 16))]

    def _check_device(self, t):
        if t.device.index != self._device:
            raise ValueError(f"tensor on {t.device}, plan built on cuda:{self._device}")

    def execute(self, f, out=None, stream=None):
        """c[W, M, N] (CUDA tensor) = DGT of f[W, L] (CUDA tensor); 1-D f gives c[M, N]."""
        import torch
        if not (isinstance(f, torch.Tensor) and f.is_cuda):
            raise TypeError("execute() takes a CUDA tensor; use execute_host() for host arrays")
        squeeze = f.dim() == 1
        f2 = f.reshape(1, -1) if squeeze else f
        want = self._rdt if self.real_input else self._cdt
        if f2.dtype != want or not f2.is_contiguous():
            raise TypeError(f"f must be a contiguous {want} tensor of shape (W, L)")
        W = f2.shape[0]
        if f2.dim() != 2 or f2.shape[1] != self.L:
            raise ValueError("f has the wrong length")
        self._check_device(f2)
        if out is None:
            out = torch.empty((W, self.M, self.N), dtype=self._cdt, device=f.device)
        elif (out.dtype != self._cdt or not out.is_contiguous() or out.numel() != W * self.M * self.N
              or out.device != f2.device):
            raise TypeError("bad output tensor")
        _check(_lib.dgt_execute(self._h, ctypes.c_void_p(f2.data_ptr()), ctypes.c_void_p(out.data_ptr()), W,
                                _stream_ptr(stream)), "dgt_execute")
        return out[0] if squeeze else out

    def inverse(self, c, out=None, stream=None):
        """f[W, L] (CUDA tensor, complex) = synthesis of c[W, M, N] (CUDA tensor) with the plan's
        window as the synthesis window (dgt_execute_inverse); 2-D c gives f[L].  A plan built
        with the canonical dual window inverts the DGT of a plan built with the window."""
        import torch
        if not (isinstance(c, torch.Tensor) and c.is_cuda):
            raise TypeError("inverse() takes a CUDA tensor")
        squeeze = c.dim() == 2
        c2 = c.reshape(1, self.M, self.N) if squeeze else c
        if c2.dtype != self._cdt or not c2.is_contiguous() or tuple(c2.shape[1:]) != (self.M, self.N):
            raise TypeError(f"c must be a contiguous {self._cdt} tensor of shape (W, M, N)")
        W = c2.shape[0]
        self._check_device(c2)
        if out is None:
            out = torch.empty((W, self.L), dtype=self._cdt, device=c.device)
        elif out.dtype != self._cdt or not out.is_contiguous() or out.numel() != W * self.L or out.device != c2.device:
            raise TypeError("bad output tensor")
        _check(_lib.dgt_execute_inverse(self._h, ctypes.c_void_p(c2.data_ptr()), ctypes.c_void_p(out.data_ptr()), W,
                                        _stream_ptr(stream)), "dgt_execute_inverse")
        return out[0] if squeeze else out

    def dual_window(self, tight: bool = False, stream=None) -> np.ndarray:
        """Canonical dual (S^{-1} g) or tight (S^{-1/2} g) window of the plan's window on its
        lattice, computed on the GPU (dgt_window_dual); returned as a host numpy array."""
        out = np.empty(self.L, dtype=self._np_c)
        _check(_lib.dgt_window_dual(self._h, 1 if tight else 0, ctypes.c_void_p(out.ctypes.data), DGT_G_ON_HOST,
                                    _stream_ptr(stream)), "dgt_window_dual")
        return out

    def execute_host(self, f, out=None, stream=None):
        """End-to-end call on HOST arrays (numpy or CPU tensors; pinned memory is faster)."""
        import torch
        want = self._rdt if self.real_input else self._cdt
        if isinstance(f, torch.Tensor):
            if f.is_cuda:
                raise TypeError("execute_host() takes host arrays; use execute() for CUDA tensors")
            squeeze = f.dim() == 1
            f2 = f.reshape(1, -1) if squeeze else f
            if f2.dtype != want or not f2.is_contiguous() or f2.dim() != 2 or f2.shape[1] != self.L:
                raise TypeError(f"f must be a contiguous {want} CPU tensor of shape (W, L)")
            fptr, W = f2.data_ptr(), f2.shape[0]
            if out is None:
                out = torch.empty((W, self.M, self.N), dtype=self._cdt, pin_memory=f2.is_pinned())
            elif (out.is_cuda or out.dtype != self._cdt or not out.is_contiguous()
                  or out.numel() != W * self.M * self.N):
                raise TypeError("bad output tensor")
            optr = out.data_ptr()
        else:
            np_want = np.dtype(str(want).replace("torch.", ""))
            f_np = np.asarray(f)
            squeeze = f_np.ndim == 1
            f2 = np.ascontiguousarray(np.atleast_2d(f_np), dtype=np_want)
            if f2.ndim != 2 or f2.shape[1] != self.L:
                raise ValueError(f"f must have shape (W, {self.L})")
            fptr, W = f2.ctypes.data, f2.shape[0]
            np_c = self._np_c
            if out is None:
                out = np.empty((W, self.M, self.N), dtype=np_c)
            elif (out.dtype != np_c or not out.flags.c_contiguous or out.size != W * self.M * self.N
                  or not out.flags.writeable):
                raise TypeError("bad output array")
            optr = out.ctypes.data
        _check(_lib.dgt_execute_host(self._h, ctypes.c_void_p(fptr), ctypes.c_void_p(optr), W, _stream_ptr(stream)),
               "dgt_execute_host")
        return out[0] if squeeze else out
