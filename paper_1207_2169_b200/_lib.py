"""ctypes binding of libgwas.so (include/gwas.h).  Argument marshalling only -- every step of the path runs in
the library's CUDA kernels.  Importing this module fails loudly if the in-tree library is missing: there is no
CPU fallback."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgwas.so")

GWAS_OK, GWAS_E_ARG, GWAS_E_NOT_SPD, GWAS_E_EIG, GWAS_E_CUDA, GWAS_E_NOMEM, GWAS_E_STATE = range(7)
STATUS_NAMES = {0: "GWAS_OK", 1: "GWAS_E_ARG", 2: "GWAS_E_NOT_SPD", 3: "GWAS_E_EIG", 4: "GWAS_E_CUDA",
                5: "GWAS_E_NOMEM", 6: "GWAS_E_STATE"}
XR_F64, XR_U8 = 0, 1
OUT_SNP, OUT_FULL = 0, 1
VAR_TEXTBOOK, VAR_LITERAL = 0, 1
PAIR_OK, PAIR_COLLINEAR, PAIR_NONFINITE = 0, 1, 2
K1, K2, K3, H2D = 0, 1, 2, 3
ALG_EIG, ALG_CHOL = 0, 1
EST_ML, EST_REML = 0, 1
NUM_TIMERS = 4

EXPORTS = ["gwas_default_options", "gwas_state_bytes", "gwas_workspace_bytes", "gwas_setup", "gwas_setup_estimate", "gwas_estimate_ms", "gwas_trait_rank", "gwas_run_info", "gwas_estimate_grid_argmax", "gwas_attach",
           "gwas_run", "gwas_timings", "gwas_kernel_times", "gwas_gemm_tn", "gwas_destroy", "gwas_last_error",
           "gwas_version"]


class GwasOptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("xr_dtype", C.c_int32), ("output_mode", C.c_int32),
                ("var_convention", C.c_int32), ("block_cols", C.c_int64), ("eps_spd", C.c_double),
                ("eps_collinear", C.c_double), ("compute_stream", C.c_void_p), ("copy_stream", C.c_void_p),
                ("timing", C.c_int32), ("int8_slices", C.c_int32),
                ("overlap", C.c_int32), ("algorithm", C.c_int32), ("fuse_k2", C.c_int32),
                ("trait_rank", C.c_int32)]


class GwasError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built -- run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, i64, i32, sz, dp = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t, C.POINTER(C.c_double)
    opt = C.POINTER(GwasOptions)
    sig = {
        "gwas_default_options": (None, [opt]),
        "gwas_state_bytes": (sz, [i64, i64, i64, opt]),
        "gwas_workspace_bytes": (sz, [i64, i64, i64, opt]),
        "gwas_setup": (C.c_int, [opt, i64, i64, i64, P, P, P, P, P, P, sz, P, sz, C.POINTER(P)]),
        "gwas_setup_estimate": (C.c_int, [opt, i64, i64, i64, P, P, P, i32, P, P, P, P, sz, P, sz, C.POINTER(P)]),
        "gwas_estimate_ms": (C.c_int, [P, dp]),
        "gwas_trait_rank": (C.c_int, [P, C.POINTER(C.c_int32), dp, dp]),
        "gwas_run_info": (C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
        "gwas_estimate_grid_argmax": (C.c_int, [P, C.POINTER(C.c_int32)]),
        "gwas_attach": (C.c_int, [opt, i64, i64, i64, P, sz, P, sz, C.POINTER(P)]),
        "gwas_run": (C.c_int, [P, i64, P, i64, P, P, P]),
        "gwas_timings": (C.c_int, [P, dp, dp, dp]),
        "gwas_kernel_times": (C.c_int, [P, dp, C.POINTER(C.c_int64), i32]),
        "gwas_gemm_tn": (C.c_int, [i64, i64, i64, P, i64, i32, P, i64, P, i64, i64, P]),
        "gwas_destroy": (None, [P]),
        "gwas_last_error": (C.c_char_p, []),
        "gwas_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(code):
    if code != GWAS_OK:
        raise GwasError(code, lib.gwas_last_error().decode())
    return code


def default_options():
    o = GwasOptions()
    lib.gwas_default_options(C.byref(o))
    return o
