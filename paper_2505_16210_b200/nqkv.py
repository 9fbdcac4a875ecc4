"""Thin ctypes binding of the NQKV C ABI (include/nqkv.h).

Argument marshalling only: every step of the hot path runs in libnqkv.so's
CUDA kernels.  PyTorch supplies device memory and the stream.  There is no
CPU fallback: if the library is missing this module raises at import time.
Function names mirror the C entry points.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

_LIB_PATH = os.environ.get("NQKV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                       "libnqkv.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the NQKV path has no CPU fallback)")
_lib = ctypes.CDLL(_LIB_PATH)

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
_fp = ctypes.POINTER(ctypes.c_float)


class KvLayout(ctypes.Structure):
    """nqkv_kv_layout (include/nqkv.h): grouped-query head mapping and the
    paged cache (readings R16, R17)."""
    _fields_ = [("kv_heads", ctypes.c_int), ("block_table", ctypes.c_void_p),
                ("pages_per_seq", ctypes.c_int), ("page_size", ctypes.c_int),
                ("n_pages", ctypes.c_int)]


_lp = ctypes.POINTER(KvLayout)

_SIGS = {
    "nqkv_abi_version": (_i32, []),
    "nqkv_status_string": (ctypes.c_char_p, [_i32]),
    "nqkv_last_error": (ctypes.c_char_p, []),
    "nqkv_levels": (_i32, [_fp]),
    "nqkv_thresholds": (_i32, [_fp]),
    "nqkv_quantize": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i32,
                             _vp, _vp, _vp]),
    "nqkv_dequantize": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "nqkv_decode_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "nqkv_decode_counter_bytes": (_sz, [_i32, _i32]),
    "nqkv_decode_attention": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                     ctypes.c_float, _vp, _vp, _sz, _vp]),
    "nqkv_decode_step": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32,
                                _i32, _i32, _i32, ctypes.c_float, _vp, _vp, _sz, _vp]),
    "nqkv_encode_normalized": (_i32, [_vp, _i64, _vp, _vp]),
    "nqkv_decode_plan_bytes": (_sz, []),
    "nqkv_decode_plan": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _sz, _vp]),
    "nqkv_decode_attention_planned": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                                             _i32, ctypes.c_float, _vp, _vp, _sz, _vp, _i32, _vp]),
    "nqkv_decode_step_planned": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                        _i32, _i32, _i32, _i32, ctypes.c_float, _vp, _vp, _sz,
                                        _vp, _i32, _vp]),
    "nqkv_decode_step_gather": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                       _i32, _i32, _i32, _i32, ctypes.c_float, _vp, _vp, _i32,
                                       _i32, _i32, ctypes.c_uint, _vp, _vp, _sz, _vp, _i32, _vp]),
    "nqkv_gather_epoch_bump": (_i32, [_vp, _vp]),
    "nqkv_gather_wait": (_i32, [_vp, _i32, _vp, _vp]),
    "nqkv_prefill_attention": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                      _i32, ctypes.c_float, _vp, _vp]),
    "nqkv_build_id": (ctypes.c_char_p, []),
    "nqkv_decode_attention_kv": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                        _lp, ctypes.c_float, _vp, _vp, _sz, _vp]),
    "nqkv_prefill_attention_kv": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                         _i32, _lp, ctypes.c_float, _vp, _vp]),
    "nqkv_quantize_pair": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i32,
                                  _vp, _vp, _vp, _vp, _vp]),
    "nqkv_quantize_kv": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _lp,
                                _vp, _vp, _vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
ABI_VERSION = 4
if _lib.nqkv_abi_version() != ABI_VERSION:
    raise ImportError("libnqkv.so ABI version mismatch; rebuild")

EARLY_START = 1     # NQKV_EARLY_START: plan and cache not written by the kernel just before

STATUS = {0: "NQKV_OK", -1: "NQKV_ERR_NULL", -2: "NQKV_ERR_SHAPE", -3: "NQKV_ERR_UNSUPPORTED",
          -4: "NQKV_ERR_ALIGN", -5: "NQKV_ERR_WORKSPACE", -6: "NQKV_ERR_CUDA",
          -7: "NQKV_ERR_INTERNAL"}


class NQKVError(RuntimeError):
    def __init__(self, status: int, where: str):
        detail = _lib.nqkv_last_error().decode() if status == -6 else ""
        super().__init__(f"{where}: {STATUS.get(status, status)} "
                         f"({_lib.nqkv_status_string(status).decode()}) {detail}".rstrip())
        self.status = status


def _check(status: int, where: str) -> None:
    if status != 0:
        raise NQKVError(status, where)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


# ----------------------------------------------------------------- host ----
def nqkv_levels() -> np.ndarray:
    out = np.zeros(16, np.float32)
    _check(_lib.nqkv_levels(out.ctypes.data_as(_fp)), "nqkv_levels")
    return out


def nqkv_thresholds() -> np.ndarray:
    out = np.zeros(15, np.float32)
    _check(_lib.nqkv_thresholds(out.ctypes.data_as(_fp)), "nqkv_thresholds")
    return out


def nqkv_decode_workspace_bytes(B: int, H: int, hd: int, Tc: int) -> int:
    return int(_lib.nqkv_decode_workspace_bytes(B, H, hd, Tc))


def nqkv_decode_counter_bytes(B: int, H: int) -> int:
    return int(_lib.nqkv_decode_counter_bytes(B, H))


SCALE_F16 = 0x10000   # NQKV_SCALE_F16: block scales stored as fp16 (lossless for fp16 inputs)


def _blkarg(blk: int, *scales: torch.Tensor) -> int:
    """blk, or blk | NQKV_SCALE_F16 when the scale tensors are fp16."""
    dt = {t.dtype for t in scales}
    assert len(dt) == 1 and dt <= {torch.float32, torch.float16}, dt
    return blk | SCALE_F16 if torch.float16 in dt else blk


# --------------------------------------------------------------- device ----
def nqkv_quantize(x: torch.Tensor, pos: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor,
                  blk: int, stream=None) -> None:
    """Append x (fp16 [B, n_new, H, hd], hd contiguous, any outer strides) at
    rows pos[b].. of the cache tensors codes [B,H,Tc,hd/2] u8 / scales
    [B,H,Tc,hd/blk] f32 or f16."""
    B, n_new, H, hd = x.shape
    Tc = codes.shape[2]
    assert x.dtype == torch.float16 and x.stride(3) == 1
    assert pos.dtype == torch.int32 and codes.dtype == torch.uint8
    assert codes.is_contiguous() and scales.is_contiguous() and tuple(codes.shape[:2]) == (B, H)
    _check(_lib.nqkv_quantize(_ptr(x), x.stride(0), x.stride(1), x.stride(2), B, H, hd, n_new,
                              _blkarg(blk, scales),
                              _ptr(pos), Tc, _ptr(codes), _ptr(scales), _stream(stream)),
           "nqkv_quantize")


def nqkv_quantize_pair(k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, k_codes: torch.Tensor,
                       k_scales: torch.Tensor, v_codes: torch.Tensor, v_scales: torch.Tensor,
                       blk: int, stream=None) -> None:
    """K and V of a layer appended in one launch (= two nqkv_quantize calls)."""
    B, n_new, H, hd = k.shape
    Tc = k_codes.shape[2]
    assert v.shape == k.shape and v.stride() == k.stride() and k.dtype == v.dtype == torch.float16
    assert k.stride(3) == 1 and pos.dtype == torch.int32
    for c, s in ((k_codes, k_scales), (v_codes, v_scales)):
        assert c.dtype == torch.uint8 and c.is_contiguous() and s.is_contiguous() and tuple(c.shape[:2]) == (B, H)
    _check(_lib.nqkv_quantize_pair(_ptr(k), _ptr(v), k.stride(0), k.stride(1), k.stride(2), B, H, hd,
                                   n_new, _blkarg(blk, k_scales, v_scales), _ptr(pos), Tc,
                                   _ptr(k_codes), _ptr(k_scales), _ptr(v_codes), _ptr(v_scales),
                                   _stream(stream)), "nqkv_quantize_pair")


def nqkv_dequantize(codes: torch.Tensor, scales: torch.Tensor, blk: int, n_tokens: int | None = None,
                    out_dtype=torch.float32, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    B, H, Tc, hb = codes.shape
    hd = hb * 2
    n_tokens = Tc if n_tokens is None else n_tokens
    if out is None:
        out = torch.empty((B, H, n_tokens, hd), dtype=out_dtype, device=codes.device)
    code = {torch.float32: 0, torch.float16: 1}[out.dtype]
    _check(_lib.nqkv_dequantize(_ptr(codes), _ptr(scales), B, H, Tc, hd, _blkarg(blk, scales),
                                n_tokens, code,
                                _ptr(out), _stream(stream)), "nqkv_dequantize")
    return out


def nqkv_decode_attention(q: torch.Tensor, k_codes: torch.Tensor, k_scales: torch.Tensor,
                          v_codes: torch.Tensor, v_scales: torch.Tensor, seq_lens: torch.Tensor,
                          blk: int, workspace: torch.Tensor, softmax_scale: float | None = None,
                          out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """out[b,h] = softmax(softmax_scale * q k^T) v over the first seq_lens[b]
    cached tokens.  workspace: zero-filled uint8 tensor of
    nqkv_decode_workspace_bytes(...) bytes (see make_workspace)."""
    B, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, H, hd), dtype=torch.float32, device=q.device)
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_decode_attention(_ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes),
                                      _ptr(v_scales), _ptr(seq_lens), B, H, hd,
                                      _blkarg(blk, k_scales, v_scales), Tc,
                                      float(softmax_scale), _ptr(out), _ptr(workspace),
                                      workspace.numel() * workspace.element_size(),
                                      _stream(stream)), "nqkv_decode_attention")
    return out


def nqkv_decode_step(k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor,
                     k_codes: torch.Tensor, k_scales: torch.Tensor, v_codes: torch.Tensor,
                     v_scales: torch.Tensor, seq_lens: torch.Tensor, blk: int,
                     workspace: torch.Tensor, softmax_scale: float | None = None,
                     out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Fused decode step: append k_new/v_new (fp16 [B, H, hd], hd contiguous)
    at row seq_lens[b]-1 and attend over seq_lens[b] tokens, one launch."""
    B, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, H, hd), dtype=torch.float32, device=q.device)
    assert k_new.shape == (B, H, hd) and v_new.shape == (B, H, hd)
    assert k_new.stride() == v_new.stride() and k_new.stride(2) == 1
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_decode_step(_ptr(k_new), _ptr(v_new), k_new.stride(0), k_new.stride(1),
                                 _ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes),
                                 _ptr(v_scales), _ptr(seq_lens), B, H, hd,
                                 _blkarg(blk, k_scales, v_scales), Tc,
                                 float(softmax_scale), _ptr(out), _ptr(workspace),
                                 workspace.numel() * workspace.element_size(), _stream(stream)),
           "nqkv_decode_step")
    return out


def nqkv_prefill_attention(q: torch.Tensor, k_codes: torch.Tensor, k_scales: torch.Tensor,
                           v_codes: torch.Tensor, v_scales: torch.Tensor, seq_lens: torch.Tensor,
                           blk: int, softmax_scale: float | None = None,
                           out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Causal prefill attention of the prompt over the dequantised cache
    (PAPER.md:213-221): q fp16 [B, T, H, hd] -> out fp32
    [B, T, H, hd]; rows >= seq_lens[b] are zero."""
    B, T, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, T, H, hd), dtype=torch.float32, device=q.device)
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_prefill_attention(_ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes),
                                       _ptr(v_scales), _ptr(seq_lens), B, H, hd,
                                       _blkarg(blk, k_scales, v_scales), Tc, T,
                                       float(softmax_scale), _ptr(out), _stream(stream)),
           "nqkv_prefill_attention")
    return out


def kv_layout(kv_heads: int = 0, block_table: torch.Tensor | None = None, page_size: int = 0,
              n_pages: int = 0) -> KvLayout:
    """nqkv_kv_layout: kv_heads (0 = as many as query heads); block_table
    int32 [B, pages_per_seq] on the device for a paged cache."""
    if block_table is not None:
        assert block_table.dtype == torch.int32 and block_table.is_contiguous()
        return KvLayout(kv_heads, block_table.data_ptr(), block_table.shape[1], page_size, n_pages)
    return KvLayout(kv_heads, None, 0, 0, 0)


def nqkv_quantize_kv(x: torch.Tensor, pos: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor,
                     blk: int, layout: KvLayout, Tc: int, stream=None) -> None:
    """nqkv_quantize into the cache `layout` describes (paged: codes
    [n_pages, H, P, hd/2], scales [n_pages, H, P, hd/blk]; Tc = the
    per-sequence capacity)."""
    B, n_new, H, hd = x.shape
    assert x.dtype == torch.float16 and x.stride(3) == 1 and pos.dtype == torch.int32
    assert codes.dtype == torch.uint8 and codes.is_contiguous() and scales.is_contiguous()
    _check(_lib.nqkv_quantize_kv(_ptr(x), x.stride(0), x.stride(1), x.stride(2), B, H, hd, n_new,
                                 _blkarg(blk, scales), _ptr(pos), Tc, ctypes.byref(layout),
                                 _ptr(codes), _ptr(scales), _stream(stream)), "nqkv_quantize_kv")


def nqkv_decode_attention_kv(q: torch.Tensor, k_codes, k_scales, v_codes, v_scales, seq_lens,
                             blk: int, layout: KvLayout, Tc: int, workspace: torch.Tensor,
                             softmax_scale: float | None = None, out: torch.Tensor | None = None,
                             stream=None) -> torch.Tensor:
    """nqkv_decode_attention over a KV layout: q [B, H, hd] (query heads),
    cache as `layout` says; Tc = the per-sequence capacity."""
    B, H, hd = q.shape
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, H, hd), dtype=torch.float32, device=q.device)
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_decode_attention_kv(_ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes),
                                         _ptr(v_scales), _ptr(seq_lens), B, H, hd,
                                         _blkarg(blk, k_scales, v_scales), Tc, ctypes.byref(layout),
                                         float(softmax_scale), _ptr(out), _ptr(workspace),
                                         workspace.numel() * workspace.element_size(),
                                         _stream(stream)), "nqkv_decode_attention_kv")
    return out


def nqkv_prefill_attention_kv(q: torch.Tensor, k_codes, k_scales, v_codes, v_scales, seq_lens,
                              blk: int, layout: KvLayout, Tc: int, softmax_scale: float | None = None,
                              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """nqkv_prefill_attention over a KV layout: q [B, T, H, hd]."""
    B, T, H, hd = q.shape
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, T, H, hd), dtype=torch.float32, device=q.device)
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_prefill_attention_kv(_ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes),
                                          _ptr(v_scales), _ptr(seq_lens), B, H, hd,
                                          _blkarg(blk, k_scales, v_scales), Tc, T,
                                          ctypes.byref(layout), float(softmax_scale), _ptr(out),
                                          _stream(stream)), "nqkv_prefill_attention_kv")
    return out


def make_plan(device="cuda") -> torch.Tensor:
    """Buffer for nqkv_decode_plan (device, caller-owned)."""
    return torch.zeros(int(_lib.nqkv_decode_plan_bytes()), dtype=torch.uint8, device=device)


def nqkv_decode_plan(seq_lens: torch.Tensor, H: int, Tc: int, fused: bool, plan: torch.Tensor,
                     stream=None, hd: int = 64) -> torch.Tensor:
    """Per-step schedule shared by every layer's planned decode call."""
    assert seq_lens.dtype == torch.int32
    _check(_lib.nqkv_decode_plan(_ptr(seq_lens), seq_lens.numel(), H, hd, Tc, int(bool(fused)),
                                 _ptr(plan), plan.numel() * plan.element_size(), _stream(stream)),
           "nqkv_decode_plan")
    return plan


def nqkv_decode_attention_planned(q, k_codes, k_scales, v_codes, v_scales, seq_lens, blk,
                                  workspace, plan, softmax_scale=None, out=None, stream=None,
                                  flags=0):
    B, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, H, hd), dtype=torch.float32, device=q.device)
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    _check(_lib.nqkv_decode_attention_planned(
        _ptr(q), _ptr(k_codes), _ptr(k_scales), _ptr(v_codes), _ptr(v_scales), _ptr(seq_lens), B, H,
        hd, _blkarg(blk, k_scales, v_scales), Tc, float(softmax_scale), _ptr(out), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _ptr(plan), int(flags), _stream(stream)),
        "nqkv_decode_attention_planned")
    return out


def nqkv_decode_step_planned(k_new, v_new, q, k_codes, k_scales, v_codes, v_scales, seq_lens, blk,
                             workspace, plan, softmax_scale=None, out=None, stream=None, flags=0):
    B, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    if out is None:
        out = torch.empty((B, H, hd), dtype=torch.float32, device=q.device)
    assert k_new.shape == (B, H, hd) and v_new.shape == (B, H, hd)
    assert k_new.stride() == v_new.stride() and k_new.stride(2) == 1
    assert q.dtype == torch.float16 and q.is_contiguous() and out.is_contiguous()
    _check(_lib.nqkv_decode_step_planned(
        _ptr(k_new), _ptr(v_new), k_new.stride(0), k_new.stride(1), _ptr(q), _ptr(k_codes),
        _ptr(k_scales), _ptr(v_codes), _ptr(v_scales), _ptr(seq_lens), B, H, hd,
        _blkarg(blk, k_scales, v_scales), Tc,
        float(softmax_scale), _ptr(out), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _ptr(plan), int(flags), _stream(stream)), "nqkv_decode_step_planned")
    return out


def nqkv_decode_step_gather(k_new, v_new, q, k_codes, k_scales, v_codes, v_scales, seq_lens, blk,
                            workspace, plan, peer_out_ptrs: torch.Tensor, peer_flag_ptrs: torch.Tensor,
                            G: int, rank: int, epoch: int = 0, epoch_ptr: torch.Tensor | None = None,
                            softmax_scale=None, stream=None, flags=0):
    """nqkv_decode_step_planned with the all-gather fused into the epilogue:
    output rows go to every rank's [B, G*H, hd] buffer (peer_out_ptrs: int64
    device tensor [G] of their addresses), then epoch is release-stored into
    flags[rank] of every rank (peer_flag_ptrs: int64 device tensor [G] of
    uint32[G] flag arrays).  epoch_ptr (int32 device scalar, read at the end
    of the launch) replaces epoch under CUDA-graph replay."""
    B, H, hd = q.shape
    Tc = k_codes.shape[2]
    if softmax_scale is None:
        softmax_scale = 1.0 / math.sqrt(hd)
    assert k_new.shape == (B, H, hd) and v_new.shape == (B, H, hd)
    assert k_new.stride() == v_new.stride() and k_new.stride(2) == 1
    assert q.dtype == torch.float16 and q.is_contiguous()
    assert peer_out_ptrs.dtype == torch.int64 and peer_flag_ptrs.dtype == torch.int64
    assert peer_out_ptrs.numel() == G and peer_flag_ptrs.numel() == G
    _check(_lib.nqkv_decode_step_gather(
        _ptr(k_new), _ptr(v_new), k_new.stride(0), k_new.stride(1), _ptr(q), _ptr(k_codes),
        _ptr(k_scales), _ptr(v_codes), _ptr(v_scales), _ptr(seq_lens), B, H, hd,
        _blkarg(blk, k_scales, v_scales), Tc, float(softmax_scale), _ptr(peer_out_ptrs),
        _ptr(peer_flag_ptrs), int(G), int(rank), int(G * H), int(epoch), _ptr(epoch_ptr), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _ptr(plan), int(flags), _stream(stream)),
        "nqkv_decode_step_gather")


def nqkv_gather_epoch_bump(epoch_ptr: torch.Tensor, stream=None) -> None:
    _check(_lib.nqkv_gather_epoch_bump(_ptr(epoch_ptr), _stream(stream)), "nqkv_gather_epoch_bump")


def nqkv_gather_wait(flags: torch.Tensor, epoch_ptr: torch.Tensor, stream=None) -> None:
    """Stream-ordered wait until every entry of flags (this rank's int32 flag
    arrays) equals *epoch_ptr (system-scope acquire)."""
    assert flags.dtype == torch.int32 and flags.is_contiguous()
    _check(_lib.nqkv_gather_wait(_ptr(flags), flags.numel(), _ptr(epoch_ptr), _stream(stream)),
           "nqkv_gather_wait")


def nqkv_encode_normalized(n: torch.Tensor, stream=None) -> torch.Tensor:
    assert n.dtype == torch.float32 and n.is_contiguous()
    codes = torch.empty(n.shape, dtype=torch.uint8, device=n.device)
    _check(_lib.nqkv_encode_normalized(_ptr(n), n.numel(), _ptr(codes), _stream(stream)),
           "nqkv_encode_normalized")
    return codes


# ------------------------------------------------------------ conveniences --
def make_workspace(B: int, H: int, hd: int, Tc: int, device="cuda") -> torch.Tensor:
    return torch.zeros(nqkv_decode_workspace_bytes(B, H, hd, Tc), dtype=torch.uint8, device=device)


def scales_shape(B: int, H: int, Tc: int, hd: int, blk: int) -> tuple:
    """[B, H, Tc, hd/blk]; blk > hd (a block spans blk/hd adjacent heads, the
    paper's blk 256): [B, H*hd/blk, Tc, 1]."""
    if blk <= hd:
        return (B, H, Tc, hd // blk)
    hpb = blk // hd
    assert H % hpb == 0, "a head shard must hold whole head groups"
    return (B, H // hpb, Tc, 1)


class KVCache:
    """Per-layer packed NF4 K/V cache in the library's layout:
    codes u8 [B,H,Tc,hd/2], scales f32 (or f16) scales_shape(...) for K and V."""

    def __init__(self, B: int, H: int, hd: int, Tc: int, blk: int = 64, device="cuda",
                 scale_dtype=torch.float32):
        """scale_dtype torch.float16 stores block scales as fp16 (lossless for
        fp16 inputs: NQKV_SCALE_F16)."""
        assert Tc % 64 == 0 and scale_dtype in (torch.float32, torch.float16)
        self.B, self.H, self.hd, self.Tc, self.blk = B, H, hd, Tc, blk
        self.k_codes = torch.zeros((B, H, Tc, hd // 2), dtype=torch.uint8, device=device)
        self.v_codes = torch.zeros_like(self.k_codes)
        self.k_scales = torch.zeros(scales_shape(B, H, Tc, hd, blk), dtype=scale_dtype, device=device)
        self.v_scales = torch.zeros_like(self.k_scales)

    def append(self, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, stream=None) -> None:
        if k.stride() == v.stride() and (k.data_ptr() - v.data_ptr()) % 32 == 0:
            nqkv_quantize_pair(k, v, pos, self.k_codes, self.k_scales, self.v_codes, self.v_scales,
                               self.blk, stream)       # one launch for K and V
        else:
            nqkv_quantize(k, pos, self.k_codes, self.k_scales, self.blk, stream)
            nqkv_quantize(v, pos, self.v_codes, self.v_scales, self.blk, stream)

    def attend(self, q: torch.Tensor, seq_lens: torch.Tensor, workspace: torch.Tensor,
               out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        return nqkv_decode_attention(q, self.k_codes, self.k_scales, self.v_codes, self.v_scales,
                                     seq_lens, self.blk, workspace, out=out, stream=stream)

    def step(self, k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor,
             seq_lens: torch.Tensor, workspace: torch.Tensor, out: torch.Tensor | None = None,
             stream=None) -> torch.Tensor:
        """Fused append + attend (seq_lens counts the appended token)."""
        return nqkv_decode_step(k_new, v_new, q, self.k_codes, self.k_scales, self.v_codes,
                                self.v_scales, seq_lens, self.blk, workspace, out=out, stream=stream)

    def attend_planned(self, q, seq_lens, workspace, plan, out=None, stream=None, flags=0):
        return nqkv_decode_attention_planned(q, self.k_codes, self.k_scales, self.v_codes,
                                             self.v_scales, seq_lens, self.blk, workspace, plan,
                                             out=out, stream=stream, flags=flags)

    def step_planned(self, k_new, v_new, q, seq_lens, workspace, plan, out=None, stream=None,
                     flags=0):
        """Fused append + attend with a per-step plan (nqkv_decode_plan, fused=True)."""
        return nqkv_decode_step_planned(k_new, v_new, q, self.k_codes, self.k_scales,
                                        self.v_codes, self.v_scales, seq_lens, self.blk,
                                        workspace, plan, out=out, stream=stream, flags=flags)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size()
                   for t in (self.k_codes, self.v_codes, self.k_scales, self.v_scales))
