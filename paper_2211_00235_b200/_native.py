"""ctypes binding of the C-ABI library (include/evo_b200.h).

This is the ONLY way the package computes: there is no CPU or PyTorch
fallback.  If the library is missing or a call fails, an exception is
raised (mapped onto the reference's error taxonomy, src/errors.py:9-38).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ContractError, DimensionError, NumericsError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libevo_b200.so")

EVO_F32, EVO_BF16 = 0, 1
EPI_NONE, EPI_RELU, EPI_SIGMOID_FROM = 0, 1, 2

c_i64, c_i32, c_f32, c_vp, c_sz = C.c_int64, C.c_int32, C.c_float, C.c_void_p, C.c_size_t


class EvoMat(C.Structure):
    _fields_ = [("ptr", c_vp), ("rs", c_i64), ("cs", c_i64), ("bs1", c_i64),
                ("bs2", c_i64), ("rdiv", c_i64), ("rs0", c_i64), ("cdiv", c_i64),
                ("cs0", c_i64)]


class GemmDesc(C.Structure):
    _fields_ = [("dtype_ab", c_i32), ("dtype_c", c_i32), ("M", c_i64), ("N", c_i64),
                ("K", c_i64), ("B1", c_i64), ("B2", c_i64), ("A", EvoMat), ("B", EvoMat),
                ("C", EvoMat), ("alpha", c_f32), ("epilogue", c_i32), ("epi_col0", c_i32),
                ("accumulate", c_i32), ("split_k", c_i32), ("bias", c_vp),
                ("residual", c_vp), ("force_simt", c_i32), ("workspace", c_vp),
                ("workspace_bytes", c_sz)]


class AttnDesc(C.Structure):
    _fields_ = [("dtype", c_i32), ("nb", c_i64), ("H", c_i32), ("L", c_i32), ("D", c_i32),
                ("scale", c_f32), ("q", c_vp), ("k", c_vp), ("v", c_vp), ("g", c_vp),
                ("sb", c_i64), ("sl", c_i64), ("o", c_vp), ("gm", c_vp), ("o_sb", c_i64),
                ("o_sl", c_i64), ("bias", c_vp), ("bh", c_i64), ("bq", c_i64),
                ("bk", c_i64), ("lse", c_vp), ("dgm", c_vp), ("dq", c_vp), ("dk", c_vp),
                ("dv", c_vp), ("dgpre", c_vp), ("dbias", c_vp), ("workspace", c_vp),
                ("workspace_bytes", c_sz), ("dgate_bias", c_vp)]


# name -> (restype, argtypes)
_SIGS = {
    "evo_gemm": (c_i32, [C.POINTER(GemmDesc), c_vp]),
    "evo_gemm_workspace_bytes": (c_sz, [C.POINTER(GemmDesc)]),
    "evo_layernorm_fwd": (c_i32, [c_i32, c_i32, c_i64, c_i32, c_vp, c_i64, c_i64, c_vp, c_vp,
                                  c_vp, c_i64, c_vp, c_vp, c_f32, c_vp]),
    "evo_layernorm_bwd": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_i32, c_vp, c_i64, c_vp, c_i64,
                                  c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                  c_i32, c_vp, c_sz, c_vp]),
    "evo_layernorm_bwd_workspace_bytes": (c_sz, [c_i64, c_i32]),
    "evo_layernorm_fwd_split": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_f32,
                                        c_vp]),
    "evo_relu_bwd_colsum": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "evo_layernorm_bwd_proj": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_sz, c_vp]),
    "evo_layernorm_bwd_ex": (c_i32, [c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                     c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "evo_attention_fwd": (c_i32, [C.POINTER(AttnDesc), c_vp]),
    "evo_attention_bwd": (c_i32, [C.POINTER(AttnDesc), c_vp]),
    "evo_attention_bwd_workspace_bytes": (c_sz, [C.POINTER(AttnDesc)]),
    "evo_reduce_lead": (c_i32, [c_i32, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i32,
                                c_vp]),
    "evo_attn_long_softmax": (c_i32, [c_i64, c_i32, c_i32, c_i64, c_vp, c_vp, c_i64, c_i64,
                                      c_i64, c_vp, c_vp, c_vp]),
    "evo_attn_flash_fwd": (c_i32, [C.POINTER(AttnDesc), c_vp]),
    "evo_attn_flash_bwd": (c_i32, [C.POINTER(AttnDesc), c_vp]),
    "evo_attn_flash_bwd_workspace_bytes": (c_sz, [C.POINTER(AttnDesc)]),
    "evo_attn_long_gate": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "evo_attn_long_prep": (c_i32, [c_i64, c_i32, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                   c_i64, c_vp, c_vp]),
    "evo_attn_long_dsoftmax": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64,
                                       c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp,
                                       c_vp, c_i32, c_vp]),
    "evo_colsum": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_i64, c_vp, c_i32, c_vp, c_sz, c_vp]),
    "evo_colsum_workspace_bytes": (c_sz, [c_i64]),
    "evo_copy2d": (c_i32, [c_i32, c_i32, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64,
                           c_vp]),
    "evo_copy3d": (c_i32, [c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp,
                           c_i64, c_i64, c_i64, c_vp]),
    "evo_zero": (c_i32, [c_vp, c_sz, c_vp]),
    "evo_mul2d": (c_i32, [c_i32, c_i32, c_i32, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp,
                          c_i64, c_vp]),
    "evo_trimul_gate_fwd": (c_i32, [c_i32, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "evo_trimul_gate_bwd": (c_i32, [c_i32, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                    c_vp, c_vp, c_sz, c_vp]),
    "evo_trimul_gate_bwd_workspace_bytes": (c_sz, [c_i64, c_i32]),
    "evo_outgate_fwd": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                c_vp]),
    "evo_outgate_bwd": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "evo_outgate_bwd_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "evo_relu_bwd": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "evo_sq_mean": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "evo_add": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "evo_div_scalar": (c_i32, [c_i64, c_vp, c_f32, c_vp, c_vp]),
    "evo_split_bf16": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                               c_vp]),
    "evo_last_error": (C.c_char_p, []),
    "evo_version": (c_i32, []),
    "evo_launch_count": (c_i64, []),
    "evo_tc_available": (c_i32, []),
    "evo_backend_count": (c_i64, [c_i32]),
    "evo_last_backend": (c_i32, []),
    "evo_set_strict_tc": (None, [c_i32]),
    "evo_get_strict_tc": (c_i32, []),
}

EXPORTED = tuple(_SIGS)

_lib = None


class NativeLibraryMissing(RuntimeError):
    """The CUDA library was not built; the package has no fallback."""


def lib():
    """Load (once) and return the ctypes handle.  Raises loudly when absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found: build it with "
                "`python -m paper_2211_00235_b200.build_lib` (nvcc, sm_100a). "
                "There is no CPU fallback.")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


_STATUS = {-1: ContractError, -2: DimensionError, -3: NumericsError, -4: RuntimeError}


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().evo_last_error().decode(errors="replace")
        raise _STATUS.get(rc, RuntimeError)(f"{what} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(lib().evo_launch_count())


# engines (include/evo_b200.h EVO_BK_*)
BACKENDS = ("gemm_tc", "gemm_simt", "gemm_skinny", "attn_tc", "attn_simt", "attn_flash")


def backend_counts() -> dict:
    """Calls served by each engine since the library was loaded."""
    L = lib()
    return {name: int(L.evo_backend_count(i)) for i, name in enumerate(BACKENDS)}


def last_backend() -> str | None:
    b = int(lib().evo_last_backend())
    return BACKENDS[b] if 0 <= b < len(BACKENDS) else None


class strict_tc:
    """Context manager for strict tensor-core mode (default ON): inside
    ``strict_tc(False)`` a bf16 GEMM / attention the tensor-core kernels do
    not take may run on the SIMT kernels instead of raising."""

    def __init__(self, on: bool = True):
        self.on = on
        self.prev = None

    def __enter__(self):
        L = lib()
        self.prev = int(L.evo_get_strict_tc())
        L.evo_set_strict_tc(1 if self.on else 0)
        return self

    def __exit__(self, *exc):
        lib().evo_set_strict_tc(self.prev)
        return False
