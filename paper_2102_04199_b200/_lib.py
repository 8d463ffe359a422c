"""ctypes binding of libkerntune_b200.so (the C-ABI in include/kerntune_b200.h).

This is the reference-side binding a maintainer would add: plain ctypes over
`extern "C"` entry points, device pointers from torch tensors, the current
torch CUDA stream passed as a void*.  There is no fallback: importing the
product API without the built library raises, and every call checks the
returned status (KT_E_* -> DomainError / NumericError).
"""

from __future__ import annotations

import ctypes
import os
import pathlib

from .errors import DomainError, NumericError

KT_F = 12
KT_MAX_KNOBS = 8
KT_MAX_AXES = 6
KT_MAX_LOOPS = 12
KT_MAX_CARD = 160
KT_MAX_LAYERS = 4
KT_MAX_DIM = 64
KT_MAX_NODES = 64

KT_OK, KT_E_SHAPE, KT_E_EMPTY, KT_E_RANGE, KT_E_UNSUPPORTED, KT_E_CUDA, KT_E_NUMERIC, KT_E_ARG = range(8)
_DOMAIN_CODES = {KT_E_SHAPE, KT_E_EMPTY, KT_E_RANGE, KT_E_UNSUPPORTED, KT_E_ARG}

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libkerntune_b200.so"

i32, i64, u32, u64, f32, f64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                ctypes.c_float, ctypes.c_double)
vp = ctypes.c_void_p


class SpecTable(ctypes.Structure):
    _fields_ = [
        ("n_knobs", i32), ("n_axes", i32), ("n_loops", i32), ("n_nodes", i32),
        ("n_pairs", i32), ("auto_knob", i32), ("expl_knob", i32), ("pad0", i32),
        ("space_size", u64),
        ("card", u32 * KT_MAX_KNOBS),
        ("axis_knob", i32 * KT_MAX_AXES),
        ("axis_reduce", i32 * KT_MAX_AXES),
        ("loop_row", i32 * KT_MAX_LOOPS),
        ("auto_vals", i32 * 4),
        ("expl_vals", i32 * 2),
        ("pad1", i32 * 2),
        ("outer", (i32 * KT_MAX_CARD) * KT_MAX_AXES),
        ("inner", (i32 * KT_MAX_CARD) * KT_MAX_AXES),
        ("raw_log2", ((f64 * KT_MAX_CARD) * KT_MAX_AXES) * 2),
        ("nrm_ext", (f32 * KT_MAX_CARD) * KT_MAX_LOOPS),
        ("nrm_log2ext", (f32 * KT_MAX_CARD) * KT_MAX_LOOPS),
        ("nrm_stride", (f32 * KT_MAX_CARD) * KT_MAX_LOOPS),
        ("nrm_const", (f32 * KT_F) * KT_MAX_LOOPS),
        ("nrm_unroll1", f32 * KT_MAX_LOOPS),
        ("fmean", f64 * KT_F),
        ("fstd", f64 * KT_F),
        ("card_magic", u64 * KT_MAX_KNOBS),
        ("digit_mult", u32 * 8),
        ("digit_card", u32 * 8),
        ("digit_mult_magic", u64 * 8),
        ("digit_card_magic", u64 * 8),
        ("choice_off", i32 * (KT_MAX_AXES + 1)),
        ("pad2", i32),
    ]


class Dims(ctypes.Structure):
    _fields_ = [
        ("F", i32), ("n_gcn", i32),
        ("gcn", i32 * (KT_MAX_LAYERS + 1)),
        ("n_head", i32),
        ("head", i32 * (KT_MAX_LAYERS + 2)),
        ("off_gcn", i32 * KT_MAX_LAYERS),
        ("off_agg", i32),
        ("off_hw", i32 * (KT_MAX_LAYERS + 1)),
        ("off_hb", i32 * (KT_MAX_LAYERS + 1)),
        ("off_head", i32),
        ("n_head_params", i32),
        ("n_params", i32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "kt_version": (ctypes.c_int, []),
    "kt_last_error": (ctypes.c_char_p, []),
    "kt_launch_count": (i64, []),
    "kt_sync_check": (ctypes.c_int, [vp]),
    "kt_encode_raw": (ctypes.c_int, [vp, vp, i64, vp, vp, vp]),
    "kt_encode_raw_choices": (ctypes.c_int, [vp, vp, i64, vp, vp, vp]),
    "kt_score_indices": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, vp, i64, i64, vp, vp, vp, vp]),
    "kt_score_indices_fp32": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, vp, i64, i64, vp, vp, vp, vp]),
    "kt_embed_csr": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp,
                                    i64, vp, vp, vp]),
    "kt_head_forward": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, i64, vp, vp]),
    "kt_gcn_layer": (ctypes.c_int, [vp, i32, vp, vp, vp, i32, i32, i32, i64, i32, vp, vp, i32, vp, vp, vp, vp, vp,
                                    i32, i32, vp, vp]),
    "kt_readout": (ctypes.c_int, [vp, i32, i64, i32, vp, vp, vp, vp]),
    "kt_grad_workspace_bytes": (i64, [ctypes.POINTER(Dims), i64]),
    "kt_grad": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, i64,
                               i32, vp, vp, f32, vp, vp, i64, vp]),
    "kt_sgd": (ctypes.c_int, [vp, vp, f32, i64, vp, vp]),
    "kt_pretrain_sgd": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp,
                                       i64, f32, vp]),
    "kt_head_loss_grad": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, i64, vp, vp, vp]),
    "kt_head_hvp": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, i64, vp, vp]),
    "kt_fine_tune": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, i64, f32, i32, vp, vp, vp]),
    "kt_maml_workspace_bytes": (i64, [ctypes.POINTER(Dims), i32, i32, i32]),
    "kt_maml_tasks": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, vp, i32, f32, i32, i32, vp, vp,
                                     vp, i64, vp]),
    "kt_maml_task_grads": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, vp, i32, f32, i32, i32, vp,
                                          vp, vp, i64, vp]),
    "kt_task_sum_update": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, i32, f32, vp, vp, vp, vp]),
    "kt_maml_step": (ctypes.c_int, [ctypes.POINTER(Dims), vp, vp, vp, vp, vp, vp, vp, i32, f32, i32, i32, f32, vp,
                                    vp, vp, i64, vp]),
    "kt_sweep_host": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, vp, i32, i64, vp, vp, i32, vp, vp, vp, vp, vp,
                                     i64, vp, vp]),
    "kt_score_indices_ex": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp]),
    "kt_score_indices_flags": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, i32,
                                              vp]),
    "kt_topk_keys": (ctypes.c_int, [vp, i64, i32, i32, vp, vp, vp, i64, vp]),
    "kt_topk_key_hist": (vp, [vp]),
    "kt_gp_gram": (ctypes.c_int, [vp, i32, vp, i32, i32, vp, vp, vp]),
    "kt_gp_factor": (ctypes.c_int, [vp, i32, i32, vp, i32, vp, ctypes.c_double, ctypes.c_double, vp, vp, vp, vp]),
    "kt_gp_workspace_bytes": (i64, [i32, i32, i32]),
    "kt_gp_posterior": (ctypes.c_int, [vp, i32, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, vp]),
    "kt_gp_ucb": (ctypes.c_int, [vp, vp, i32, ctypes.c_double, ctypes.c_double, i32, vp, vp, i64, vp]),
    "kt_sa_propose": (ctypes.c_int, [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "kt_sa_accept": (ctypes.c_int, [i32, i32, vp, vp, f64, vp, vp, vp, vp]),
    "kt_sa_draws": (ctypes.c_int, [vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "kt_sa_run": (ctypes.c_int, [vp, ctypes.POINTER(Dims), vp, i32, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                 vp, vp, vp]),
    "kt_topk_workspace_bytes": (i64, [i64, i32]),
    "kt_topk": (ctypes.c_int, [vp, vp, i64, i64, vp, i64, i32, vp, vp, vp, i64, vp]),
    "kt_topk_merge": (ctypes.c_int, [vp, vp, i64, i32, vp, vp, vp, i64, vp]),
}

_lib = None


def exported_symbols() -> list:
    return sorted(_SIGS)


def load(path: str | os.PathLike | None = None):
    """Load (once) and type the library.  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise NumericError(
            f"{p} is missing: build it with `python -m paper_2102_04199_b200.build` "
            "(there is no CPU fallback for the cost-model path)")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == KT_OK:
        return
    msg = load().kt_last_error().decode(errors="replace")
    text = f"{what}: {msg} (status {rc})"
    if rc in _DOMAIN_CODES:
        raise DomainError(text)
    raise NumericError(text)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL; an int is already an address)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream
