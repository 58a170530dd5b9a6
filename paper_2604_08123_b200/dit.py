"""Thin ctypes binding of libdit.so (include/dit.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used
only to own device memory and streams.  There is no CPU fallback: if the
shared library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DIT_LIB_OVERRIDE") or os.path.join(_HERE, "libdit.so")   # override: perf experiments only
_lib = None

DIT_OK = 0
ERRORS = {0: "DIT_OK", 1: "DIT_EINVAL", 2: "DIT_ENOMEM", 3: "DIT_ECUDA", 4: "DIT_EEXIST", 5: "DIT_ERANK",
          6: "DIT_ENOSPC", 7: "DIT_ENOENT", 8: "DIT_EBATCH", 9: "DIT_ESHAPE", 10: "DIT_EADAPTER",
          11: "DIT_EALIAS", 12: "DIT_EPARALLEL", 13: "DIT_ENCCL", 14: "DIT_ENOWEIGHTS"}
CODES = {v: k for k, v in ERRORS.items()}


class dit_config(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("heads", C.c_int32), ("depth_double", C.c_int32),
                ("depth_single", C.c_int32), ("in_channels", C.c_int32), ("txt_dim", C.c_int32),
                ("pooled_dim", C.c_int32), ("mlp_ratio", C.c_int32), ("rope_axes", C.c_int32 * 3),
                ("rope_theta", C.c_float), ("guidance_embed", C.c_int32), ("max_batch", C.c_int32),
                ("max_img_tokens", C.c_int32), ("max_txt_tokens", C.c_int32), ("max_rank", C.c_int32),
                ("max_adapters", C.c_int32), ("arch", C.c_int32), ("qk_norm", C.c_int32),
                ("pos_embed_max", C.c_int32), ("pos_embed_base", C.c_int32), ("max_sp_world", C.c_int32)]


ARCH = {"flux": 0, "sd3": 1}


class dit_tensor(C.Structure):
    _fields_ = [("name", C.c_char_p), ("ptr", C.c_void_p), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("shape", C.c_int64 * 4)]


class dit_batch(C.Structure):
    _fields_ = [("batch", C.c_int32), ("img_h", C.c_int32), ("img_w", C.c_int32), ("txt_tokens", C.c_int32),
                ("adapter_id", C.POINTER(C.c_int32)), ("sigma", C.POINTER(C.c_float)),
                ("sigma_next", C.POINTER(C.c_float)), ("guidance", C.POINTER(C.c_float)),
                ("cn_scale", C.POINTER(C.c_float)), ("latents_in", C.c_void_p), ("latents_out", C.c_void_p),
                ("txt", C.c_void_p), ("pooled", C.c_void_p), ("v_out", C.c_void_p),
                ("cfg_scale", C.POINTER(C.c_float)), ("img_hw", C.POINTER(C.c_int32))]


EXPORTS = {
    "dit_workspace_bytes": (C.c_size_t, [C.POINTER(dit_config)]),
    "dit_create": (C.c_int, [C.POINTER(dit_config), C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "dit_destroy": (None, [C.c_void_p]),
    "dit_last_error": (C.c_char_p, [C.c_void_p]),
    "dit_load_weights": (C.c_int, [C.c_void_p, C.POINTER(dit_tensor), C.c_int]),
    "lora_register": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.POINTER(dit_tensor), C.c_int,
                                C.c_void_p]),
    "lora_unregister": (C.c_int, [C.c_void_p, C.c_int32]),
    "dit_merge_bytes": (C.c_size_t, [C.POINTER(dit_config)]),
    "lora_merge": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p]),
    "lora_unmerge": (C.c_int, [C.c_void_p]),
    "lora_merge_inplace": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64),
                                     C.c_void_p]),
    "controlnet_inject": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_float, C.c_void_p]),
    "controlnet_clear": (C.c_int, [C.c_void_p]),
    "controlnet_inject_flag": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_float, C.c_void_p,
                                         C.c_uint32]),
    "dit_debug_delayed_publish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32, C.c_uint64,
                                            C.c_void_p]),
    "dit_debug_host_delay": (C.c_int, [C.c_void_p, C.c_uint64]),
    "controlnet_push": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32, C.c_void_p]),
    "dit_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dit_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dit_ipc_close": (C.c_int, [C.c_void_p]),
    "sp_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "lp_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "lp_init_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "dit_peer_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sp_init_peers": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "lp_init_peers": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "dit_step": (C.c_int, [C.c_void_p, C.POINTER(dit_batch), C.c_void_p]),
    "dit_graph_create": (C.c_int, [C.c_void_p, C.POINTER(dit_batch), C.c_void_p, C.POINTER(C.c_void_p)]),
    "dit_graph_launch": (C.c_int, [C.c_void_p, C.POINTER(dit_batch), C.c_void_p]),
    "dit_graph_destroy": (None, [C.c_void_p]),
    "dit_step_flops": (C.c_double, [C.c_void_p, C.POINTER(dit_batch)]),
    "dit_last_launch_count": (C.c_int, [C.c_void_p]),
    "dit_sp_exchange": (C.c_int, [C.c_void_p]),
    "dit_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "dit_profile_read": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int)]),
    "dit_profile_reset": (C.c_int, [C.c_void_p]),
    "dit_fill_synthetic": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint64, C.c_uint64, C.c_float, C.c_float,
                                     C.c_void_p]),
    "dit_local_group_create": (C.c_void_p, [C.c_int32]),
    "dit_local_group_destroy": (None, [C.c_void_p]),
    "sp_init_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "dit_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "dit_debug_attention_trace": (C.c_int, [C.c_void_p]),
    "dit_debug_attention_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "dit_debug_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                 C.c_void_p]),
    "dit_debug_gemm_resid": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                       C.c_int32, C.c_int32, C.c_void_p]),
    "dit_debug_attention": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_void_p, C.c_void_p]),
    "dit_sp_layout": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_int64), C.c_int64]),
    "dit_debug_row_adapter": (C.c_int, [C.c_void_p, C.POINTER(dit_batch), C.POINTER(C.c_int32), C.c_int]),
    "dit_debug_plan": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int]),
    "dit_debug_shard_map": (C.c_int, [C.c_void_p, C.POINTER(dit_batch), C.POINTER(C.c_int32), C.c_int]),
}


def load_library():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdit.so not found at {LIB_PATH}: the CUDA extension is not built "
                           "(run `python __graft_entry__.py`); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        if os.environ.get("DIT_LIB_OVERRIDE") and not hasattr(lib, name):
            continue   # an older experimental build (perf comparisons only)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class DitError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _check(code, ctx=None):
    if code != DIT_OK:
        lib = load_library()
        msg = lib.dit_last_error(ctx).decode() if lib else ""
        raise DitError(code, msg)


def make_config(cfg, max_batch, max_img_tokens, max_txt_tokens, max_rank=0, max_adapters=0,
                max_sp_world=0) -> dit_config:
    c = dit_config()
    c.hidden, c.heads = cfg.hidden, cfg.heads
    c.depth_double, c.depth_single = cfg.depth_double, cfg.depth_single
    c.in_channels, c.txt_dim, c.pooled_dim = cfg.in_channels, cfg.txt_dim, cfg.pooled_dim
    c.mlp_ratio = cfg.mlp_ratio
    for i in range(3):
        c.rope_axes[i] = cfg.rope_axes[i]
    c.rope_theta = cfg.rope_theta
    c.guidance_embed = int(cfg.guidance_embed)
    c.max_batch, c.max_img_tokens, c.max_txt_tokens = max_batch, max_img_tokens, max_txt_tokens
    c.max_rank, c.max_adapters = max_rank, max_adapters
    c.arch = ARCH[getattr(cfg, "arch", "flux")]
    c.qk_norm = int(getattr(cfg, "qk_norm", True))
    c.pos_embed_max = getattr(cfg, "pos_embed_max", 192)
    c.pos_embed_base = getattr(cfg, "pos_embed_base", 64)
    c.max_sp_world = max_sp_world
    return c


def tensor_desc(name: str, t) -> dit_tensor:
    """dit_tensor for a torch bf16 CUDA tensor (keeps `name` bytes alive via the struct)."""
    d = dit_tensor()
    d.name = name.encode()
    d.ptr = t.data_ptr()
    d.dtype = 0
    d.rank = t.dim()
    for i, s in enumerate(t.shape):
        d.shape[i] = s
    return d


def _arr(ctype, vals):
    a = (ctype * len(vals))(*vals)
    return a


class DiT:
    """One context (one GPU): borrowed weights, adapter pool, ControlNet slots."""

    def __init__(self, cfg, max_batch, max_img_tokens, max_txt_tokens, max_rank=0, max_adapters=0, device=0,
                 max_sp_world=0):
        import torch
        self.lib = load_library()
        self.cfg = cfg
        self.device = device
        self.c_cfg = make_config(cfg, max_batch, max_img_tokens, max_txt_tokens, max_rank, max_adapters, max_sp_world)
        nbytes = self.lib.dit_workspace_bytes(C.byref(self.c_cfg))
        if nbytes == 0:
            raise DitError(1, "invalid config")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        ctx = C.c_void_p()
        _check(self.lib.dit_create(C.byref(self.c_cfg), device, self.workspace.data_ptr(), nbytes, C.byref(ctx)))
        self.ctx = ctx
        self.weights: Dict[str, object] = {}
        self._keep = []

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dit_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- boundary calls (same names as include/dit.h)
    def dit_load_weights(self, tensors: Dict[str, object]):
        descs = (dit_tensor * len(tensors))(*[tensor_desc(k, v) for k, v in tensors.items()])
        _check(self.lib.dit_load_weights(self.ctx, descs, len(tensors)), self.ctx)
        self.weights.update(tensors)

    def lora_register(self, adapter_id: int, rank: int, scale: float, tensors: Dict[str, object], stream=None):
        descs = (dit_tensor * len(tensors))(*[tensor_desc(k, v) for k, v in tensors.items()])
        _check(self.lib.lora_register(self.ctx, adapter_id, rank, scale, descs, len(tensors),
                                      self._stream(stream)), self.ctx)

    def lora_unregister(self, adapter_id: int):
        _check(self.lib.lora_unregister(self.ctx, adapter_id), self.ctx)

    def merge_bytes(self) -> int:
        return int(self.lib.dit_merge_bytes(C.byref(self.c_cfg)))

    def lora_merge(self, adapter_id: int, merged=None, stream=None):
        """Patch `adapter_id` into a copy of the adapted weights (caller-owned `merged`, a uint8
        device tensor of >= merge_bytes(); allocated here if None and kept until lora_unmerge)."""
        import torch
        if merged is None:
            merged = torch.empty(self.merge_bytes() + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        ptr = merged.data_ptr()
        pad = (-ptr) % 256
        self._merged = merged
        _check(self.lib.lora_merge(self.ctx, adapter_id, C.c_void_p(ptr + pad), merged.numel() - pad,
                                   self._stream(stream)), self.ctx)

    def lora_merge_inplace(self, adapter_id: int, undo=None, stream=None) -> int:
        """Hot-patch `adapter_id` over the base weights; `undo`: a device tensor (8-byte aligned) for the
        undo log.  Returns the entries used.  With undo=None the log is sized by a first call that
        returns DIT_ENOMEM with the count, then allocated here (kept until lora_unmerge)."""
        import torch
        n = C.c_uint64(0)
        if undo is None:
            r = self.lib.lora_merge_inplace(self.ctx, adapter_id, None, 0, C.byref(n), self._stream(stream))
            if r == 0:
                self._undo = None
                return 0
            if r != 2:
                _check(r, self.ctx)
            undo = torch.empty(max(1, n.value), dtype=torch.int64, device=f"cuda:{self.device}")
        self._undo = undo
        _check(self.lib.lora_merge_inplace(self.ctx, adapter_id, C.c_void_p(undo.data_ptr()),
                                           undo.numel() * undo.element_size(), C.byref(n), self._stream(stream)),
               self.ctx)
        return n.value

    def lora_unmerge(self):
        _check(self.lib.lora_unmerge(self.ctx), self.ctx)
        self._merged = None

    def controlnet_inject(self, slot: int, block: int, residual, scale: float = 1.0, ready_event=None):
        self._keep.append(residual)
        ev = ready_event.cuda_event if ready_event is not None else None
        _check(self.lib.controlnet_inject(self.ctx, slot, block, residual.data_ptr(), scale, ev), self.ctx)

    def controlnet_inject_flag(self, slot: int, block: int, residual, flag, expect: int, scale: float = 1.0):
        """Deferred residual published by a device flag (a uint32 device tensor; *flag >= expect)."""
        self._keep += [residual, flag]
        _check(self.lib.controlnet_inject_flag(self.ctx, slot, block, residual.data_ptr(), scale, flag.data_ptr(),
                                               expect), self.ctx)

    def sp_init(self, world: int, rank: int, nccl_uid: Optional[bytes] = None):
        buf = C.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
        _check(self.lib.sp_init(self.ctx, world, rank, buf), self.ctx)

    def sp_init_local(self, group, rank: int):
        _check(self.lib.sp_init_local(self.ctx, group, rank), self.ctx)

    def lp_init(self, world: int, rank: int, nccl_uid: bytes):
        buf = C.create_string_buffer(nccl_uid, 128)
        _check(self.lib.lp_init(self.ctx, world, rank, buf), self.ctx)

    def peer_handle(self) -> bytes:
        """dit_peer_handle: this context's workspace handle (resets its arrival flags)."""
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        _check(self.lib.dit_peer_handle(self.ctx, buf), self.ctx)
        return buf.raw

    def sp_init_peers(self, world: int, rank: int, handles):
        """handles: every rank's peer_handle() in rank order (any transport)."""
        blob = b"".join(handles)
        _check(self.lib.sp_init_peers(self.ctx, world, rank, C.create_string_buffer(blob, len(blob))), self.ctx)

    def lp_init_peers(self, world: int, rank: int, handles):
        blob = b"".join(handles)
        _check(self.lib.lp_init_peers(self.ctx, world, rank, C.create_string_buffer(blob, len(blob))), self.ctx)

    def sp_exchange(self) -> int:
        return int(self.lib.dit_sp_exchange(self.ctx))

    def lp_init_local(self, group, rank: int):
        _check(self.lib.lp_init_local(self.ctx, group, rank), self.ctx)

    def make_batch(self, batch_size, img_h, img_w, txt_tokens, adapter_id, sigma, sigma_next, guidance,
                   latents_in, latents_out, txt, pooled, v_out=None, cn_scale=None, cfg_scale=None,
                   img_hw=None) -> dit_batch:
        b = dit_batch()
        b.batch, b.img_h, b.img_w, b.txt_tokens = batch_size, img_h, img_w, txt_tokens
        keep = [_arr(C.c_int32, [int(x) for x in adapter_id]), _arr(C.c_float, [float(x) for x in sigma]),
                _arr(C.c_float, [float(x) for x in sigma_next]), _arr(C.c_float, [float(x) for x in guidance])]
        b.adapter_id, b.sigma, b.sigma_next, b.guidance = keep
        if cn_scale is not None:
            cs = _arr(C.c_float, [float(x) for x in cn_scale])
            keep.append(cs)
            b.cn_scale = cs
        if cfg_scale is not None:
            gs = _arr(C.c_float, [float(x) for x in cfg_scale])
            keep.append(gs)
            b.cfg_scale = gs
        if img_hw is not None:
            hw = _arr(C.c_int32, [int(x) for pair in img_hw for x in pair])
            keep.append(hw)
            b.img_hw = hw
        b.latents_in, b.latents_out = latents_in.data_ptr(), latents_out.data_ptr()
        b.txt, b.pooled = txt.data_ptr(), pooled.data_ptr()
        b.v_out = v_out.data_ptr() if v_out is not None else None
        b._keep = keep
        return b

    def dit_step(self, batch: dit_batch, stream=None):
        _check(self.lib.dit_step(self.ctx, C.byref(batch), self._stream(stream)), self.ctx)

    def graph_create(self, batch: dit_batch, stream=None):
        """Capture one dit_step on `batch` (dit_graph_create); returns the graph handle."""
        g = C.c_void_p()
        _check(self.lib.dit_graph_create(self.ctx, C.byref(batch), self._stream(stream), C.byref(g)), self.ctx)
        return g

    def graph_launch(self, graph, batch: dit_batch, stream=None):
        _check(self.lib.dit_graph_launch(graph, C.byref(batch), self._stream(stream)), self.ctx)

    def graph_destroy(self, graph):
        self.lib.dit_graph_destroy(graph)

    def step_flops(self, batch: dit_batch) -> float:
        return float(self.lib.dit_step_flops(self.ctx, C.byref(batch)))

    def last_launch_count(self) -> int:
        return int(self.lib.dit_last_launch_count(self.ctx))

    def profile(self, enable: bool):
        _check(self.lib.dit_profile(self.ctx, int(enable)), self.ctx)

    def profile_read(self, kind: int):
        ms, fl, n = C.c_double(), C.c_double(), C.c_int()
        _check(self.lib.dit_profile_read(self.ctx, kind, C.byref(ms), C.byref(fl), C.byref(n)), self.ctx)
        return ms.value, fl.value, n.value

    def profile_reset(self):
        _check(self.lib.dit_profile_reset(self.ctx), self.ctx)

    def debug_row_adapter(self, batch: dit_batch, cap: int):
        out = (C.c_int32 * cap)()
        n = self.lib.dit_debug_row_adapter(self.ctx, C.byref(batch), out, cap)
        if n < 0:
            raise DitError(-n, "debug_row_adapter")
        return list(out[:n])

    def debug_plan(self, which: int, kind: int, cap: int = 1 << 20):
        out = (C.c_int32 * cap)()
        n = self.lib.dit_debug_plan(self.ctx, which, kind, out, cap)
        if n < 0:
            raise DitError(-n, "debug_plan")
        return list(out[:n])

    def debug_shard_map(self, batch: dit_batch, cap: int):
        out = (C.c_int32 * cap)()
        n = self.lib.dit_debug_shard_map(self.ctx, C.byref(batch), out, cap)
        if n < 0:
            raise DitError(-n, "debug_shard_map")
        return list(out[:n])

    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)


IPC_HANDLE_BYTES = 72
PEER_HANDLE_BYTES = 80


def ipc_export(t) -> bytes:
    """Inter-process handle of a device tensor's first byte (dit_ipc_export)."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    _check(load_library().dit_ipc_export(t.data_ptr(), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    out = C.c_void_p()
    _check(load_library().dit_ipc_open(C.create_string_buffer(handle, IPC_HANDLE_BYTES), C.byref(out)))
    return out.value


def ipc_close(ptr: int):
    _check(load_library().dit_ipc_close(C.c_void_p(ptr)))


def controlnet_push(dst: int, src, flag: int, value: int, stream=None):
    """Producer side of the deferred ControlNet input: copy `src` (a device tensor) to the
    consumer's buffer `dst` (a device pointer, e.g. from ipc_open) and release *flag = value."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(load_library().controlnet_push(C.c_void_p(dst), C.c_void_p(src.data_ptr()), src.numel() * src.element_size(),
                                          C.c_void_p(flag), value, C.c_void_p(s.cuda_stream)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load_library().dit_nccl_unique_id(buf))
    return buf.raw


def sp_layout(which, world, rank, B, H, Nt, Ni):
    """Host copy of the SP index maps used by the kernels (see include/dit.h)."""
    import numpy as np
    lib = load_library()
    cap = 3 * B * H * (Nt + Ni) * max(world, 1) + 16
    out = (C.c_int64 * cap)()
    n = lib.dit_sp_layout(which, world, rank, B, H, Nt, Ni, out, cap)
    if n < 0:
        raise DitError(-n, "sp_layout")
    return np.frombuffer(out, dtype=np.int64, count=n).copy()


def fill_synthetic(t, seed: int, tensor_id: int, scale: float, offset: float, stream=None):
    """Device-side counter generator (bit-identical to synth.counter_bf16_bits)."""
    import torch
    lib = load_library()
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib.dit_fill_synthetic(t.data_ptr(), t.numel(), seed, tensor_id, scale, offset, s.cuda_stream))
