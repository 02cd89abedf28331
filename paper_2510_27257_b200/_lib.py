"""ctypes binding of libstp.so (include/stp.h, include/stp_ops.h).

Argument marshalling only: every step of the path runs in the library's
kernels.  Loading fails loudly if libstp.so is missing (there is no
fallback); build it with `python -m paper_2510_27257_b200.build`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstp.so")


class StpError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn} -> {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libstp.so not built at {LIB_PATH}; run python -m paper_2510_27257_b200.build")
    return C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)


lib = _load()

i32, i64, f32, vp, cp = C.c_int32, C.c_int64, C.c_float, C.c_void_p, C.c_char_p


class Action(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "chunk", "f_mb", "b_mb", "w_mb", "w_chunk")]


class Unit(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("action", "stream", "op", "layer", "chunk", "mb", "dep0", "dep1")]


class ModelCfg(C.Structure):
    _fields_ = [("vocab", i32), ("hidden", i32), ("n_layers", i32), ("n_q_heads", i32),
                ("n_kv_heads", i32), ("head_dim", i32), ("ffn", i32), ("seq", i32),
                ("rms_eps", f32), ("rope_theta", f32), ("qkv_bias", i32), ("dtype", i32)]


class ParallelCfg(C.Structure):
    _fields_ = [("tp", i32), ("pp", i32), ("vpp", i32), ("n_micro", i32), ("tp_rank", i32),
                ("pp_rank", i32), ("layers_per_vstage", C.POINTER(C.c_int32)), ("sched_kind", i32)]


class VitCfg(C.Structure):
    _fields_ = [("hidden", i32), ("n_layers", i32), ("n_heads", i32), ("head_dim", i32), ("mlp", i32),
                ("patch_dim", i32), ("grid_h", i32), ("grid_w", i32), ("ln_eps", f32), ("rope_theta", f32)]


class StepStats(C.Structure):
    _fields_ = [("step_ms", C.c_double), ("exposed_tp_ms", C.c_double), ("pp_bubble_ms", C.c_double),
                ("compute_busy_ms", C.c_double), ("peak_act_bytes", i64), ("n_units", i32),
                ("n_kernels", i32)]


_SIGS = {
    "stp_last_error": (cp, []),
    "stp_version": (cp, []),
    "stp_num_sms": (i32, []),
    "stp_kernel_launches": (i64, []),
    # schedule
    "stp_build_schedule": (i32, [i32, i32, i32, i32, i32, C.POINTER(vp)]),
    "stp_schedule_actions": (i32, [vp, i32, C.POINTER(Action), i32, C.POINTER(i32)]),
    "stp_schedule_units": (i32, [vp, i32, C.POINTER(i32), C.POINTER(Unit), i32, C.POINTER(i32)]),
    "stp_schedule_serialize": (i32, [vp, C.POINTER(i32), C.c_char_p, i64, C.POINTER(i64)]),
    "stp_schedule_units_mllm": (i32, [vp, i32, C.POINTER(i32), C.POINTER(Unit), i32, C.POINTER(i32)]),
    "stp_schedule_serialize_mllm": (i32, [vp, C.POINTER(i32), C.c_char_p, i64, C.POINTER(i64)]),
    "stp_schedule_stash_slots": (i32, [vp, i32, C.POINTER(i32)]),
    "stp_free_schedule": (None, [vp]),
    "stp_layer_split": (i32, [i32, i32, C.POINTER(i32)]),
    # stage
    "stp_nccl_id_bytes": (i32, []),
    "stp_nccl_get_id": (i32, [vp]),
    "stp_init_stage": (i32, [C.POINTER(ModelCfg), C.POINTER(ParallelCfg), vp, i32, C.POINTER(vp)]),
    "stp_init_stage_mllm": (i32, [C.POINTER(ModelCfg), C.POINTER(VitCfg), C.POINTER(ParallelCfg), vp, i32,
                                  C.POINTER(vp)]),
    "stp_stage_bind_images": (i32, [vp, vp]),
    "stp_stage_param_count": (i32, [vp, C.POINTER(i32)]),
    "stp_stage_param_info": (i32, [vp, i32, C.POINTER(cp), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "stp_bind_params": (i32, [vp, i32, C.POINTER(vp), C.POINTER(vp)]),
    "stp_stage_set_timing": (i32, [vp, i32]),
    "stp_train_step": (i32, [vp, vp, vp, C.POINTER(f32), C.POINTER(StepStats), vp]),
    "stp_train_step_host": (i32, [vp, vp, vp, C.POINTER(f32), C.POINTER(StepStats), vp]),
    "stp_stage_trace": (i32, [vp, C.POINTER(Unit), i32, C.POINTER(i32)]),
    "stp_stage_unit_times": (i32, [vp, C.POINTER(f32), C.POINTER(f32), i32, C.POINTER(i32)]),
    "stp_destroy_stage": (None, [vp]),
    # ops
    "stp_op_gemm": (i32, [i32, i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, vp, i64, i32, vp]),
    "stp_op_rmsnorm_fwd": (i32, [i32, i64, i64, vp, vp, vp, vp, f32, vp, vp, vp]),
    "stp_op_rmsnorm_bwd": (i32, [i32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "stp_op_rope": (i32, [i32, i32, i64, i64, i64, i32, i32, f32, i64, vp, vp]),
    "stp_op_swiglu_fwd": (i32, [i32, i64, i64, vp, vp, vp]),
    "stp_op_swiglu_bwd": (i32, [i32, i64, i64, vp, vp, vp, vp]),
    "stp_op_attn_fwd": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, i64, vp, i64, vp, vp]),
    "stp_op_attn_bwd_ws_bytes": (i64, [i64, i32, i32, i32]),
    "stp_op_attn_bwd": (i32, [i32, i64, i32, i32, i32, vp, vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, i64, vp, vp]),
    "stp_op_attn_full_fwd": (i32, [i32, i64, i32, i32, vp, i64, vp, i64, vp, vp]),
    "stp_op_attn_full_bwd": (i32, [i32, i64, i32, i32, vp, i64, vp, i64, vp, vp, vp, i64, vp, vp]),
    "stp_op_layernorm_fwd": (i32, [i32, i64, i64, vp, vp, vp, vp, vp, f32, vp, vp, vp, vp]),
    "stp_op_layernorm_bwd": (i32, [i32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "stp_op_act_fwd": (i32, [i32, i32, i64, vp, vp, vp]),
    "stp_op_act_bwd": (i32, [i32, i32, i64, vp, vp, vp, vp]),
    "stp_op_rope2d": (i32, [i32, i32, i64, i64, i64, i32, i32, i32, f32, vp, vp]),
    "stp_op_embed_fwd": (i32, [i32, i64, i64, vp, i64, i64, vp, vp, vp]),
    "stp_op_embed_bwd": (i32, [i32, i64, i64, vp, i64, i64, vp, vp, vp]),
    "stp_op_ce_stats": (i32, [i32, i64, i64, vp, i64, vp, i64, vp, vp]),
    "stp_op_lm_head_ce_ws_bytes": (i64, [i64, i64]),
    "stp_op_lm_head_ce": (i32, [i32, i64, i64, i64, vp, vp, vp, vp, i64, vp, vp, vp]),
    "stp_op_ce_combine": (i32, [i64, i32, vp, vp, vp, f32, vp]),
    "stp_op_ce_grad": (i32, [i32, i64, i64, vp, i64, vp, i64, vp, f32, vp]),
    "stp_op_colsum_acc": (i32, [i32, i64, i64, vp, i64, vp, vp]),
    "stp_op_convert": (i32, [i32, i32, i64, vp, vp, vp]),
    "stp_set_option": (i32, [cp, i64]),
    "stp_prof_enable": (i32, [i32]),
    "stp_prof_reset": (i32, []),
    "stp_prof_read": (i32, [i32, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                            C.POINTER(C.c_double)]),
}

MISSING = []
for _name, (_res, _args) in _SIGS.items():
    try:
        _f = getattr(lib, _name)
    except AttributeError:
        MISSING.append(_name)
        continue
    _f.restype = _res
    _f.argtypes = _args


def last_error() -> str:
    return lib.stp_last_error().decode()


def check(fn: str, code: int):
    if code != 0:
        raise StpError(fn, code, last_error())


def call(fn: str, *args):
    """Call an stp_* status-returning function; raise StpError on failure."""
    check(fn, getattr(lib, fn)(*args))
