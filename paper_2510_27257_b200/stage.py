"""Python binding of one STP stage (stp_init_stage / stp_bind_params /
stp_train_step).  Marshalling only: torch allocates device memory for the
parameters and fp32 gradients and supplies the process group used to
broadcast the NCCL unique id; every step of the path runs inside libstp.so.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L

SCHED = {"stp": 0, "1f1b-i": 1, "zb": 2, "stp-nobraid": 3, "stp-nosep": 4, "1f1b-i-naive": 5, "1f1b": 6,
         "stp-mem": 7}
DTYPES = {"f32": (0, torch.float32), "bf16": (1, torch.bfloat16)}


def nccl_id() -> bytes:
    n = L.lib.stp_nccl_id_bytes()
    buf = C.create_string_buffer(n)
    L.call("stp_nccl_get_id", buf)
    return buf.raw


def broadcast_nccl_id(group=None) -> Optional[bytes]:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    obj = [nccl_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def pack_vit_param(name: str, PV: Dict[str, np.ndarray], vit, tp: int, r: int) -> np.ndarray:
    """Rank r's shard of ViT / merger parameter `name` (include/stp.h MLLM
    layout): wqkv rows = [q heads of rank | k heads | v heads] (+ bqkv),
    w1 / merger.w1 row blocks (+ biases), wo / w2 / merger.w2 column blocks;
    LayerNorms, row-parallel biases and the patch embedding replicated."""
    if name.startswith("merger."):
        short = name.split(".", 1)[1]
        m4l = 4 * vit.hidden // tp
        if short in ("w1", "b1"):
            return PV[name][r * m4l:(r + 1) * m4l]
        if short == "w2":
            return PV[name][:, r * m4l:(r + 1) * m4l]
        return PV[name]
    if name == "vit.patch":
        return PV[name]
    short = name.rsplit(".", 1)[1]
    hv, nl = vit.hidden, vit.n_heads // tp * vit.head_dim
    ml = vit.mlp // tp
    if short in ("wqkv", "bqkv"):
        w = PV[name]
        return np.concatenate([w[j * hv + r * nl:j * hv + (r + 1) * nl] for j in range(3)], 0)
    if short == "wo":
        return PV[name][:, r * nl:(r + 1) * nl]
    if short in ("w1", "b1"):
        return PV[name][r * ml:(r + 1) * ml]
    if short == "w2":
        return PV[name][:, r * ml:(r + 1) * ml]
    return PV[name]   # ln*_g / ln*_b / bo / b2


def pack_rank_param(name: str, P: Dict[str, np.ndarray], cfg, tp: int, r: int) -> np.ndarray:
    """Rank r's shard of parameter `name` in the stage layout of include/stp.h
    (fused QKV / gate-up rows, row-parallel column blocks, vocab row blocks,
    replicated gammas)."""
    d = cfg.head_dim
    qh, kh, fi, vl = cfg.n_q_heads // tp, cfg.n_kv_heads // tp, cfg.ffn // tp, cfg.vocab // tp
    if name in ("embed", "lm_head"):
        return P[name][r * vl:(r + 1) * vl]
    if name == "final_ln":
        return P[name]
    pre, short = name.rsplit(".", 1)
    pre += "."
    q_rows = slice(r * qh * d, (r + 1) * qh * d)
    k_rows = slice(r * kh * d, (r + 1) * kh * d)
    f_rows = slice(r * fi, (r + 1) * fi)
    if short in ("ln1", "ln2"):
        return P[name]
    if short == "wqkv":
        return np.concatenate([P[pre + "wq"][q_rows], P[pre + "wk"][k_rows], P[pre + "wv"][k_rows]], 0)
    if short == "bqkv":
        return np.concatenate([P[pre + "bq"][q_rows], P[pre + "bk"][k_rows], P[pre + "bv"][k_rows]], 0)
    if short == "wo":
        return P[pre + "wo"][:, q_rows]
    if short == "wgu":
        return np.concatenate([P[pre + "wg"][f_rows], P[pre + "wu"][f_rows]], 0)
    if short == "wd":
        return P[pre + "wd"][:, f_rows]
    raise KeyError(name)


class Stage:
    def __init__(self, cfg, tp: int = 1, pp: int = 1, n_micro: int = 1, tp_rank: int = 0, pp_rank: int = 0,
                 dtype: str = "bf16", sched: str = "stp", layers_per_vstage: Optional[Sequence[int]] = None,
                 device: int = 0, world_nccl_id: Optional[bytes] = None, vit=None,
                 offload_alpha: Optional[float] = None):
        """vit (stp_inputs.VitShape): MLLM stage, virtual stage 0 = ViT + merger
        (stp_init_stage_mllm); bind the patches with bind_images().
        offload_alpha: activation offloading (§4.3; the library reads
        STP_OFFLOAD_ALPHA at init): fraction of chunk 0's layers whose MLP
        activations go to pinned host memory between forward and backward."""
        import os
        if offload_alpha is not None:
            os.environ["STP_OFFLOAD_ALPHA"] = str(offload_alpha)
        self.cfg, self.tp, self.pp, self.m = cfg, tp, pp, n_micro
        self.vit = vit
        self.tp_rank, self.pp_rank, self.device = tp_rank, pp_rank, device
        self.dtype_code, self.torch_dtype = DTYPES[dtype]
        self.sched = sched
        vpp = 1 if sched == "1f1b" else 2
        mc = L.ModelCfg(cfg.vocab, cfg.hidden, cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim,
                        cfg.ffn, cfg.seq, cfg.rms_eps, cfg.rope_theta, int(cfg.qkv_bias), self.dtype_code)
        self._lay = None
        lay_ptr = None
        if layers_per_vstage is not None:
            self._lay = (C.c_int32 * len(layers_per_vstage))(*layers_per_vstage)
            lay_ptr = C.cast(self._lay, C.POINTER(C.c_int32))
        pc = L.ParallelCfg(tp, pp, vpp, n_micro, tp_rank, pp_rank, lay_ptr, SCHED[sched])
        self.h = C.c_void_p()
        idbuf = C.create_string_buffer(world_nccl_id, len(world_nccl_id)) if world_nccl_id else None
        torch.cuda.set_device(device)
        if vit is None:
            L.call("stp_init_stage", C.byref(mc), C.byref(pc), idbuf, device, C.byref(self.h))
        else:
            vc = L.VitCfg(vit.hidden, vit.n_layers, vit.n_heads, vit.head_dim, vit.mlp, vit.patch_dim, vit.grid_h,
                          vit.grid_w, vit.ln_eps, vit.rope_theta)
            L.call("stp_init_stage_mllm", C.byref(mc), C.byref(vc), C.byref(pc), idbuf, device, C.byref(self.h))
        if offload_alpha is not None:
            del os.environ["STP_OFFLOAD_ALPHA"]
        n = C.c_int32()
        L.call("stp_stage_param_count", self.h, C.byref(n))
        self.names: List[str] = []
        self.params: List[torch.Tensor] = []
        self.grads: List[torch.Tensor] = []
        for i in range(n.value):
            nm, numel, d0, d1 = C.c_char_p(), C.c_int64(), C.c_int64(), C.c_int64()
            L.call("stp_stage_param_info", self.h, i, C.byref(nm), C.byref(numel), C.byref(d0), C.byref(d1))
            shape = (d0.value,) if d1.value == 1 else (d0.value, d1.value)
            self.names.append(nm.value.decode())
            self.params.append(torch.zeros(shape, dtype=self.torch_dtype, device=f"cuda:{device}"))
            self.grads.append(torch.zeros(shape, dtype=torch.float32, device=f"cuda:{device}"))
        pp_ = (C.c_void_p * n.value)(*[t.data_ptr() for t in self.params])
        gp_ = (C.c_void_p * n.value)(*[t.data_ptr() for t in self.grads])
        L.call("stp_bind_params", self.h, n.value, pp_, gp_)

    def load_params(self, P: Dict[str, np.ndarray], PV: Optional[Dict[str, np.ndarray]] = None):
        for name, t in zip(self.names, self.params):
            if name.startswith(("vit.", "merger.")):
                a = pack_vit_param(name, PV, self.vit, self.tp, self.tp_rank)
            else:
                a = pack_rank_param(name, P, self.cfg, self.tp, self.tp_rank)
            t.copy_(torch.from_numpy(np.ascontiguousarray(a)))

    def bind_images(self, patches: torch.Tensor):
        """patches: device [n_micro, grid_h * grid_w, patch_dim] in the stage dtype (kept referenced)."""
        assert patches.dtype == self.torch_dtype and patches.is_contiguous()
        self._patches = patches
        L.call("stp_stage_bind_images", self.h, patches.data_ptr())

    def zero_grads(self):
        for g in self.grads:
            g.zero_()

    def set_timing(self, on: bool):
        L.call("stp_stage_set_timing", self.h, int(on))

    def step(self, tokens: Optional[torch.Tensor], targets: Optional[torch.Tensor]):
        loss = C.c_float()
        st = L.StepStats()
        L.call("stp_train_step", self.h, tokens.data_ptr() if tokens is not None else None,
               targets.data_ptr() if targets is not None else None, C.byref(loss), C.byref(st),
               torch.cuda.current_stream(self.device).cuda_stream)
        return loss.value, st

    def step_host(self, tokens: Optional[np.ndarray], targets: Optional[np.ndarray]):
        loss = C.c_float()
        st = L.StepStats()
        tk = np.ascontiguousarray(tokens, dtype=np.int32) if tokens is not None else None
        tg = np.ascontiguousarray(targets, dtype=np.int32) if targets is not None else None
        L.call("stp_train_step_host", self.h, tk.ctypes.data if tk is not None else None,
               tg.ctypes.data if tg is not None else None, C.byref(loss), C.byref(st),
               torch.cuda.current_stream(self.device).cuda_stream)
        return loss.value, st

    def trace(self):
        n = C.c_int32()
        L.lib.stp_stage_trace(self.h, None, 0, C.byref(n))
        buf = (L.Unit * max(1, n.value))()
        L.call("stp_stage_trace", self.h, buf, n.value, C.byref(n))
        return [(u.action, u.stream, u.op, u.layer, u.chunk, u.mb, u.dep0, u.dep1) for u in buf[:n.value]]

    def unit_times(self):
        n = C.c_int32()
        L.lib.stp_stage_unit_times(self.h, None, None, 0, C.byref(n))
        a = (C.c_float * max(1, n.value))()
        b = (C.c_float * max(1, n.value))()
        L.call("stp_stage_unit_times", self.h, a, b, n.value, C.byref(n))
        return list(a[:n.value]), list(b[:n.value])

    def grads_numpy(self) -> Dict[str, np.ndarray]:
        return {n: g.double().cpu().numpy() for n, g in zip(self.names, self.grads)}

    def close(self):
        if self.h:
            L.lib.stp_destroy_stage(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def schedule_units(kind: str, pp: int, n_micro: int, tp: int, pp_rank: int, layers_per_vstage: Sequence[int],
                   mllm: bool = False):
    """stp_build_schedule + stp_schedule_units (stp_schedule_units_mllm) for
    one rank (tuples in the canonical U-line field order)."""
    fn = "stp_schedule_units_mllm" if mllm else "stp_schedule_units"
    vpp = 1 if kind == "1f1b" else 2
    h = C.c_void_p()
    L.call("stp_build_schedule", pp, vpp, tp, n_micro, SCHED[kind], C.byref(h))
    try:
        lay = (C.c_int32 * len(layers_per_vstage))(*layers_per_vstage)
        n = C.c_int32()
        getattr(L.lib, fn)(h, pp_rank, lay, None, 0, C.byref(n))
        buf = (L.Unit * max(1, n.value))()
        L.call(fn, h, pp_rank, lay, buf, n.value, C.byref(n))
        return [(u.action, u.stream, u.op, u.layer, u.chunk, u.mb, u.dep0, u.dep1) for u in buf[:n.value]]
    finally:
        L.lib.stp_free_schedule(h)
