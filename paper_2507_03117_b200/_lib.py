"""ctypes binding of libblast_b200.so (C ABI declared in include/blast.h).

This module is the only place the package touches the native library. There is
no CPU fallback: if the library is missing or cannot be loaded the import of
any compute function raises, and every compute call needs CUDA tensors.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["BLAST_LIB"]) if os.environ.get("BLAST_LIB") else _HERE / "libblast_b200.so"  # BLAST_LIB: A/B builds (dev)

F32, BF16, F64 = 0, 1, 2
ACT = {"none": 0, "relu": 1, "gelu": 2, "silu": 3}

OK, EINVAL, EMISMATCH, EGRID, ECUDA, ENOMEM = range(6)

vp = C.c_void_p
i64 = C.c_int64
i32 = C.c_int32


class BcscDesc(C.Structure):
    _fields_ = [
        ("rows", i64), ("cols", i64), ("block", i32), ("dtype", i32), ("nnzb", i64),
        ("col_ptr", vp), ("row_idx", vp), ("values", vp),
        ("tf32_fwd_hi", vp), ("tf32_fwd_lo", vp), ("tf32_rt_hi", vp), ("tf32_rt_lo", vp),
        ("kmap", vp),
        ("fwd_step_ptr", vp), ("fwd_steps", vp), ("fwd_flags", vp),
        ("rt_step_ptr", vp), ("rt_steps", vp), ("rt_flags", vp),
    ]


class MlpPlanDesc(C.Structure):
    _fields_ = [
        ("gu_step_ptr", vp), ("gu_steps", vp), ("gu_flags", vp),
        ("dx_step_ptr", vp), ("dx_steps", vp), ("dx_flags", vp),
    ]


TP_MAX = 8


class TpDesc(C.Structure):
    """include/blast.h blast_tp_t"""
    _fields_ = [
        ("n", C.c_int32), ("rank", C.c_int32), ("epoch", C.c_uint32), ("reserved", C.c_int32),
        ("recv", vp * TP_MAX), ("flags", vp * TP_MAX), ("y", vp * TP_MAX), ("done", vp * TP_MAX),
    ]


# name -> (restype, argtypes)
_PROTOS = {
    "blast_last_error": (C.c_char_p, []),
    "blast_version": (C.c_int, []),
    "blast_num_sms": (C.c_int, []),
    "blast_kmap_from_bcsc": (C.c_int, [vp, vp, i64, i64, vp, vp]),
    "blast_build_plan": (C.c_int, [vp, vp, i64, i64, C.c_int, vp, vp, vp, vp]),
    "blast_balanced_schedule": (C.c_int, [vp, vp, i32, i32, i32, i32, vp, vp]),
    "blast_split_tf32": (C.c_int, [vp, vp, vp, i64, vp]),
    "blast_tf32_prepare": (C.c_int, [vp, i64, i32, vp, vp, vp, vp, vp]),
    "blast_bspmm": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.c_int, vp, vp]),
    "blast_bspmm_rt": (C.c_int, [vp, i64, C.POINTER(BcscDesc), vp, vp]),
    "blast_bspmm_ex": (C.c_int, [vp, i64, C.POINTER(BcscDesc), vp, C.c_int, vp, vp, vp]),
    "blast_bspmm_rt_act": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.c_int, vp, vp, vp]),
    "blast_activation": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, vp]),
    "blast_mlp_forward": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.POINTER(BcscDesc),
                                    C.POINTER(BcscDesc), C.POINTER(MlpPlanDesc), vp, vp, vp, vp,
                                    vp]),
    "blast_column_sums": (C.c_int, [vp, C.c_int, i64, i64, vp, vp]),
    "blast_tp_down_allreduce": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.POINTER(TpDesc), vp]),
    "blast_tp_mlp_forward": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.POINTER(BcscDesc),
                                       C.POINTER(BcscDesc), C.POINTER(MlpPlanDesc),
                                       C.POINTER(TpDesc), vp]),
    "blast_tp_wait": (C.c_int, [vp, C.c_uint32, vp]),
    "blast_mlp_forward_host": (C.c_int, [vp, i64, C.POINTER(BcscDesc), C.POINTER(BcscDesc),
                                         C.POINTER(BcscDesc), C.POINTER(MlpPlanDesc), vp, i64,
                                         vp]),
    "blast_mlp_gate_up":(C.c_int, [vp, i64, C.POINTER(BcscDesc), C.POINTER(BcscDesc),
                                    C.POINTER(MlpPlanDesc), vp, vp, vp, vp]),
    "blast_mlp_backward_dgrad": (C.c_int, [vp, i64, vp, vp, C.POINTER(BcscDesc),
                                           C.POINTER(BcscDesc), C.POINTER(BcscDesc),
                                           C.POINTER(MlpPlanDesc), vp, vp, vp, vp]),
    "blast_block_wgrad": (C.c_int, [vp, vp, i64, i64, i64, i32, C.c_int, vp, vp, i64, vp, vp,
                                    vp]),
    "blast_wgrad_plan": (C.c_int, [vp, i64, i64, i32, vp, vp, vp]),
    "blast_block_wgrad_planned": (C.c_int, [vp, vp, i64, i64, i64, i32, C.c_int, vp, vp, i64,
                                            vp, vp, vp, vp]),
    "blast_generate_masks": (C.c_int, [vp, C.c_int, vp, C.c_int, i64, i64, i32, i64, vp, vp, vp,
                                       vp, vp, vp, vp]),
    "blast_block_norms": (C.c_int, [vp, vp, i64, i64, i32, C.c_int, vp, vp, vp]),
    "blast_topk_mask": (C.c_int, [vp, i64, i64, i64, vp, vp]),
    "blast_topk_mask2": (C.c_int, [vp, vp, i64, i64, i64, vp, vp, vp]),
    "blast_mask_difference": (C.c_int, [vp, vp, i64, vp, vp, vp]),
    "blast_repack_index": (C.c_int, [vp, vp, vp, i64, i64, i32, C.c_int, vp, vp, vp]),
    "blast_repack_rows": (C.c_int, [vp, vp, i64, i64, vp, vp]),
    "blast_apply_mask_gather": (C.c_int, [vp, i64, i64, i32, C.c_int, vp, vp, C.c_int, vp, vp,
                                          vp, C.c_int, vp]),
    "blast_sgd_step": (C.c_int, [vp, vp, i64, C.c_float, vp]),
    "blast_sumsq_f64": (C.c_int, [vp, i64, C.c_int, vp, vp]),
}

EXPORTED = tuple(_PROTOS)

_lib = None


def load():
    """Load the native library (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        try:
            from . import build as _build
            _build.build(verbose=False)
        except Exception as exc:  # no silent fallback: report why the product path is gone
            raise RuntimeError(f"libblast_b200.so missing and could not be built: {exc}") from exc
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class BlastError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = load().blast_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (EINVAL, EMISMATCH, EGRID):
        raise ValueError(text)
    raise BlastError(text)


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return BF16
    if dt == torch.float32:
        return F32
    raise ValueError(f"unsupported dtype {dt}; expected float32 or bfloat16")


def require_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("blast kernels need CUDA tensors (no CPU fallback)")
