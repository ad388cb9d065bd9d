"""Python API over libgwas.so: torch provides device memory and streams; the C-ABI does all the work.

    eng = Gwas(n, p, t, device=0)                 # sizes fixed per context
    eng.setup(Phi, XL, Y, h2, sigma2)             # Alg. 4 lines 1-2, 4, 6-11
    b, var, status = eng.run(XR)                  # Alg. 4 line 3 + lines 13-16

Arrays follow the paper's shapes: Phi (n, n), XL (n, p), Y (n, t), h2 / sigma2 (t,), and X_R given SNP-major as
(ncols, ld) -- i.e. the column-major n x ncols matrix of the paper with leading dimension ld >= n (uint8 dosages or
float64).  Results are (ncols, t) [SNP i][trait j] torch tensors on the device ((ncols, t, p+1) in full mode).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

_XR = {"u8": _lib.XR_U8, "f64": _lib.XR_F64}
_OUT = {"snp": _lib.OUT_SNP, "full": _lib.OUT_FULL}
_VAR = {"textbook": _lib.VAR_TEXTBOOK, "literal": _lib.VAR_LITERAL}
_ALG = {"eig": _lib.ALG_EIG, "chol": _lib.ALG_CHOL}
_EST = {"ml": _lib.EST_ML, "reml": _lib.EST_REML}


def _ptr(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.data_ptr()
    return x.ctypes.data


def _colmajor_f64(x, device=None):
    """Return an object whose memory is x (2-D, rows x cols) in column-major fp64 order, plus its keep-alive."""
    if isinstance(x, torch.Tensor):
        t = x.to(dtype=torch.float64)
        t = t.t().contiguous() if t.dim() == 2 else t.contiguous()
        return t
    a = np.asarray(x, dtype=np.float64)
    return np.asfortranarray(a) if a.ndim == 2 else np.ascontiguousarray(a)


class Gwas:
    """One CLAK-Eig context bound to one CUDA device (include/gwas.h)."""

    def __init__(self, n: int, p: int, t: int, *, device: int = 0, xr_dtype: str = "u8", output_mode: str = "snp",
                 var_convention: str = "textbook", block_cols: int = 8192, timing: bool = False,
                 eps_spd: float = 1e-10, eps_collinear: float = 1e-10, compute_stream=None, copy_stream=None,
                 int8_slices: int = 0, overlap: bool = False, algorithm: str = "eig", fuse_k2: bool = True,
                 trait_rank: int = 0):
        self.n, self.p, self.t = int(n), int(p), int(t)
        self.w = self.p + 1
        self.device = torch.device("cuda", device)
        self.xr_dtype = xr_dtype
        self.output_mode = output_mode
        self.compute_stream = compute_stream or torch.cuda.current_stream(self.device)
        self.copy_stream = copy_stream or torch.cuda.Stream(self.device)
        o = _lib.default_options()
        o.device = device
        o.xr_dtype = _XR[xr_dtype]
        o.output_mode = _OUT[output_mode]
        o.var_convention = _VAR[var_convention]
        o.block_cols = int(block_cols)
        o.eps_spd = float(eps_spd)
        o.eps_collinear = float(eps_collinear)
        o.compute_stream = self.compute_stream.cuda_stream
        o.copy_stream = self.copy_stream.cuda_stream
        o.timing = 1 if timing else 0
        o.int8_slices = int(int8_slices)
        o.overlap = 1 if overlap else 0
        o.algorithm = _ALG[algorithm]
        o.fuse_k2 = 1 if fuse_k2 else 0
        o.trait_rank = int(trait_rank)
        self.opt = o
        self.state_bytes = lib.gwas_state_bytes(self.n, self.p, self.t, C.byref(o))
        if self.state_bytes == 0:
            raise _lib.GwasError(_lib.GWAS_E_ARG, lib.gwas_last_error().decode())
        self.work_bytes = lib.gwas_workspace_bytes(self.n, self.p, self.t, C.byref(o))
        if self.work_bytes == 0:
            raise _lib.GwasError(_lib.GWAS_E_CUDA, lib.gwas_last_error().decode())
        self.state = torch.empty(self.state_bytes, dtype=torch.uint8, device=self.device)
        self.work = torch.empty(self.work_bytes, dtype=torch.uint8, device=self.device)
        self._ctx = C.c_void_p()
        self._keep = []

    # ------------------------------------------------------------------ setup / attach
    def setup(self, Phi, XL, Y, h2, sigma2):
        """Rank-0 setup (eig + precompute) into self.state.  Inputs may be numpy or torch (host or device)."""
        self._close_ctx()
        phi = _colmajor_f64(Phi)
        xl = _colmajor_f64(XL)
        y = _colmajor_f64(np.asarray(Y).reshape(self.n, self.t) if not isinstance(Y, torch.Tensor) else Y.reshape(self.n, self.t))
        hh = _colmajor_f64(h2)
        ss = _colmajor_f64(sigma2)
        for a, shape in ((phi, (self.n, self.n)), (xl, (self.n, self.p)), (hh, (self.t,)), (ss, (self.t,))):
            if tuple(a.shape) != shape and tuple(a.shape)[::-1] != shape:
                raise ValueError(f"bad input shape {tuple(a.shape)}, expected {shape}")
        with torch.cuda.device(self.device):
            check(lib.gwas_setup(C.byref(self.opt), self.n, self.p, self.t, _ptr(phi), _ptr(xl), _ptr(y), _ptr(hh),
                                 _ptr(ss), self.state.data_ptr(), self.state_bytes, self.work.data_ptr(),
                                 self.work_bytes, C.byref(self._ctx)))
        return self

    def setup_estimate(self, Phi, XL, Y, method: str = "reml"):
        """The paper's first step + setup: estimate (h2_j, sigma2_j) per trait by ML / REML in the
        eigenbasis, then precompute with them.  Returns dict(h2, sigma2, loglik) as float64 numpy arrays (t,) and g_star (int32, the first grid argmax)."""
        self._close_ctx()
        phi = _colmajor_f64(Phi)
        xl = _colmajor_f64(XL)
        y = _colmajor_f64(np.asarray(Y).reshape(self.n, self.t) if not isinstance(Y, torch.Tensor) else Y.reshape(self.n, self.t))
        for a, shape in ((phi, (self.n, self.n)), (xl, (self.n, self.p))):
            if tuple(a.shape) != shape and tuple(a.shape)[::-1] != shape:
                raise ValueError(f"bad input shape {tuple(a.shape)}, expected {shape}")
        h2 = np.empty(self.t)
        s2 = np.empty(self.t)
        ll = np.empty(self.t)
        with torch.cuda.device(self.device):
            check(lib.gwas_setup_estimate(C.byref(self.opt), self.n, self.p, self.t, _ptr(phi), _ptr(xl), _ptr(y),
                                          _EST[method], h2.ctypes.data, s2.ctypes.data, ll.ctypes.data,
                                          self.state.data_ptr(), self.state_bytes, self.work.data_ptr(),
                                          self.work_bytes, C.byref(self._ctx)))
        gs = np.empty(self.t, dtype=np.int32)
        check(lib.gwas_estimate_grid_argmax(self._ctx, gs.ctypes.data_as(C.POINTER(C.c_int32))))
        return {"h2": h2, "sigma2": s2, "loglik": ll, "g_star": gs}

    def trait_rank(self):
        """(r, s0, s_r): the low-rank trait-weight rank chosen at setup (0 = exact weights) and the singular values."""
        r, s0, sr = C.c_int32(), C.c_double(), C.c_double()
        check(lib.gwas_trait_rank(self._ctx, C.byref(r), C.byref(s0), C.byref(sr)))
        return r.value, s0.value, sr.value

    def run_info(self):
        """{"block_cols": k used by gwas_run (resolves block_cols=0, auto), "fused_k2": K2 in K1's epilogue}."""
        k, f = C.c_int64(), C.c_int32()
        check(lib.gwas_run_info(self._ctx, C.byref(k), C.byref(f)))
        return {"block_cols": k.value, "fused_k2": bool(f.value)}

    def estimate_ms(self) -> float:
        ms = C.c_double()
        check(lib.gwas_estimate_ms(self._ctx, C.byref(ms)))
        return ms.value

    def attach(self):
        """Non-setup ranks: self.state was filled by a broadcast; validate it and create the context."""
        self._close_ctx()
        torch.cuda.synchronize(self.device)
        check(lib.gwas_attach(C.byref(self.opt), self.n, self.p, self.t, self.state.data_ptr(), self.state_bytes,
                              self.work.data_ptr(), self.work_bytes, C.byref(self._ctx)))
        return self

    # ------------------------------------------------------------------ hot path
    def alloc_outputs(self, ncols: int, host: bool = False):
        """(b, var, status) buffers: on the device, or in pinned host memory (host=True) -- then gwas_run streams
        each block's results back while later blocks compute."""
        per = (self.w,) if self.output_mode == "full" else ()
        kw = dict(pin_memory=True) if host else dict(device=self.device)
        b = torch.empty((ncols, self.t) + per, dtype=torch.float64, **kw)
        v = torch.empty((ncols, self.t) + per, dtype=torch.float64, **kw)
        s = torch.empty((ncols, self.t), dtype=torch.int8, **kw)
        return b, v, s

    def run(self, XR, ldx: int | None = None, ncols: int | None = None, out=None):
        """X_R (ncols, ld) SNP-major: torch cuda tensor, or pinned host torch tensor (staged on copy_stream).
        Returns (b, var, status) -- device tensors, or the pinned host tensors passed as `out`; asynchronous on
        compute_stream."""
        if not self._ctx:
            raise _lib.GwasError(_lib.GWAS_E_STATE, "setup()/attach() first")
        if isinstance(XR, np.ndarray):
            XR = torch.from_numpy(XR).pin_memory()
        want = torch.uint8 if self.xr_dtype == "u8" else torch.float64
        if XR.dtype != want:
            raise TypeError(f"X_R dtype {XR.dtype}, context expects {want}")
        if XR.dim() != 2 or XR.stride(1) != 1:
            raise ValueError("X_R must be (ncols, ld) with unit inner stride")
        ncols = XR.shape[0] if ncols is None else int(ncols)
        ldx = XR.stride(0) if ldx is None else int(ldx)
        if out is None:
            out = self.alloc_outputs(ncols)
        b, v, s = out
        self._keep = [XR, b, v, s]
        check(lib.gwas_run(self._ctx, ncols, XR.data_ptr(), ldx, b.data_ptr(), v.data_ptr(), s.data_ptr()))
        return b, v, s

    # ------------------------------------------------------------------ timing
    def timings(self):
        e, pcm, r = C.c_double(), C.c_double(), C.c_double()
        check(lib.gwas_timings(self._ctx, C.byref(e), C.byref(pcm), C.byref(r)))
        return {"ms_eig": e.value, "ms_precompute": pcm.value, "ms_run": r.value}

    def kernel_times(self, reset: bool = False):
        ms = (C.c_double * _lib.NUM_TIMERS)()
        n = (C.c_int64 * _lib.NUM_TIMERS)()
        check(lib.gwas_kernel_times(self._ctx, ms, n, 1 if reset else 0))
        names = ["K1", "K2", "K3", "H2D"]
        return {names[k]: {"ms": ms[k], "launches": n[k]} for k in range(_lib.NUM_TIMERS)}

    # ------------------------------------------------------------------ teardown
    def _close_ctx(self):
        if self._ctx:
            lib.gwas_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def close(self):
        self._close_ctx()

    def __del__(self):
        try:
            self._close_ctx()
        except Exception:
            pass


def gemm_tn(A: torch.Tensor, B: torch.Tensor, nsq: int | None = None, K: int | None = None) -> torch.Tensor:
    """K1/K2 kernel unit entry: C[i, c] = sum_r A[i, r] * B[c, r] (A (M, ldA) uint8 or float64, B (N, ldB) float64,
    both row-per-column on the device); columns c >= nsq use A^2.  Returns C (M, N) float64."""
    M, N = A.shape[0], B.shape[0]
    K = A.shape[1] if K is None else K
    ldc = N + (N & 1)
    C_ = torch.empty((M, ldc), dtype=torch.float64, device=A.device)
    nsq = N if nsq is None else nsq
    check(lib.gwas_gemm_tn(M, N, K, A.data_ptr(), A.stride(0), 1 if A.dtype == torch.uint8 else 0, B.data_ptr(),
                           B.stride(0), C_.data_ptr(), ldc, nsq, torch.cuda.current_stream(A.device).cuda_stream))
    return C_[:, :N]
