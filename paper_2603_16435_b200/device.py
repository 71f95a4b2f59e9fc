"""Batched, device-resident entry points over torch CUDA tensors.

These are thin wrappers over the C-ABI (include/vqkv_c.h): they validate
shapes, allocate outputs with torch's caching allocator and enqueue the
library's kernels on the current torch stream.  Nothing here computes on the
CPU.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch

from . import _lib
from .codebook import CodebookStack, DeviceStack
from .errors import InvalidInput

DEFAULT_SEARCH_BLOCK = 4096


def _dev(stack) -> DeviceStack:
    return stack.device if isinstance(stack, CodebookStack) else stack


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _need(t: torch.Tensor, dtype, name):
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise InvalidInput(f"{name} must be a contiguous CUDA {dtype} tensor")


def _pair_stride(t: torch.Tensor, dtype, name: str, inner: int) -> int:
    """Per-pair stride of a [pairs, n, D] view (in rows) or a [pairs, bytes] view (in bytes)
    whose per-pair part is contiguous.  A [pairs, capacity] payload buffer reports its
    capacity, so callers may pass a buffer longer than the payload."""
    if t.dtype != dtype:
        raise InvalidInput(f"{name} must be {dtype}")
    if not t.is_cuda:
        raise InvalidInput(f"{name} must be a CUDA tensor")
    if t.numel() == 0:
        return 0
    if t.dim() not in (2, 3):
        raise InvalidInput(f"{name} must be [pairs, rows, D] or [pairs, bytes]")
    if t.is_contiguous() or (t.shape[0] == 1 and t[0].is_contiguous()):  # dense; one pair has no real stride
        return t.shape[1]
    if t.dim() == 3:
        ok = t.stride(2) == 1 and t.stride(1) == t.shape[2] and t.stride(0) % t.shape[2] == 0
        ok = ok and t.stride(0) >= t.shape[1] * t.shape[2]
        if not ok:
            raise InvalidInput(f"{name}: rows of each pair must be contiguous")
        return t.stride(0) // t.shape[2]
    if t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        return t.stride(0)
    raise InvalidInput(f"{name}: each pair's bytes must be contiguous")


def payload_bytes(stack, rows: int) -> int:
    return _dev(stack).payload_bytes(rows)


def quantize_streams(
    stack,
    xs: torch.Tensor,
    search_block: int = DEFAULT_SEARCH_BLOCK,
    payload: Optional[torch.Tensor] = None,
    norms: Optional[torch.Tensor] = None,
    residuals: bool = False,
):
    """quantize_batch over xs [n_streams, rows, D] -> (payload [n_streams, pb] u8, norms [n_streams, rows])."""
    dev = _dev(stack)
    if xs.dim() == 2:
        xs = xs.unsqueeze(0)
    _need(xs, torch.float32, "xs")
    ns, rows, d = xs.shape
    if rows > 0 and d != dev.dim:
        raise InvalidInput(f"vector dimension {d} does not match stack dimension {dev.dim}")
    pb = dev.payload_bytes(rows)
    if payload is None:
        payload = torch.empty((ns, pb), dtype=torch.uint8, device=xs.device)
    if norms is None:
        norms = torch.empty((ns, rows), dtype=torch.float32, device=xs.device)
    res = torch.empty_like(xs) if residuals else None
    _lib.call(
        "vqkv_quantize_batch_ex", dev.h, xs.data_ptr(), ns, rows, search_block, payload.data_ptr(),
        norms.data_ptr(), res.data_ptr() if res is not None else None, _stream(xs),
    )
    return (payload, norms, res) if residuals else (payload, norms)


def quantize_streams_host(stack, xs_host: torch.Tensor, search_block: int = DEFAULT_SEARCH_BLOCK,
                          payload_host: Optional[torch.Tensor] = None, norms_host: Optional[torch.Tensor] = None,
                          blocking: bool = True):
    """quantize_batch with host (ideally pinned) buffers: H2D, encode, D2H inside the call.

    blocking=False returns once the work is queued on the current stream; the host
    buffers hold the results after that stream synchronizes (and must stay alive)."""
    dev = _dev(stack)
    if xs_host.dim() == 2:
        xs_host = xs_host.unsqueeze(0)
    if xs_host.is_cuda or xs_host.dtype != torch.float32 or not xs_host.is_contiguous():
        raise InvalidInput("xs_host must be a contiguous host float32 tensor")
    ns, rows, d = xs_host.shape
    pb = dev.payload_bytes(rows)
    if payload_host is None:
        payload_host = torch.empty((ns, pb), dtype=torch.uint8, pin_memory=xs_host.is_pinned())
    if norms_host is None:
        norms_host = torch.empty((ns, rows), dtype=torch.float32, pin_memory=xs_host.is_pinned())
    s = torch.cuda.current_stream(torch.device("cuda", dev.device)).cuda_stream
    _lib.call(
        "vqkv_quantize_batch_host" if blocking else "vqkv_quantize_batch_host_async", dev.h, xs_host.data_ptr(), ns,
        rows, search_block, payload_host.data_ptr(), norms_host.data_ptr(), s,
    )
    return payload_host, norms_host


def reconstruct_streams(stack, payload: torch.Tensor, rows: int, begin: int = 0, end: Optional[int] = None,
                        out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """reconstruct_block over each stream's payload -> [n_streams, end-begin, D] fp32."""
    dev = _dev(stack)
    end = rows if end is None else end
    if payload.dim() == 1:
        payload = payload.unsqueeze(0)
    stride = _pair_stride(payload, torch.uint8, "payload", 1)  # capacity buffers may be strided
    ns = payload.shape[0]
    if begin > end or end > rows or begin < 0:
        raise InvalidInput(f"row range [{begin}, {end}) out of bounds for {rows} rows")
    if out is None:
        out = torch.empty((ns, end - begin, dev.dim), dtype=torch.float32, device=payload.device)
    else:
        _need(out, torch.float32, "out")
        if out.numel() != ns * (end - begin) * dev.dim:
            raise InvalidInput("out must hold n_streams x (end - begin) x D floats")
    _lib.call("vqkv_reconstruct_block_ex", dev.h, payload.data_ptr(), stride, ns, rows, begin, end, out.data_ptr(),
              _stream(payload))
    return out


GM_ALIGN = 16  # group-major capacity granule (tokens)


def keycodes_gm_bytes(kstack, cap: int) -> int:
    """Bytes per pair of the group-major key-code layout for `cap` tokens (0: unsupported stack)."""
    return int(_lib.load().vqkv_keycodes_gm_bytes(_dev(kstack).h, cap))


def keycodes_to_gm(kstack, payload: torch.Tensor, count: int, gm: Optional[torch.Tensor] = None, cap: int = 0,
                   src_row: int = 0, dst_row: int = 0) -> torch.Tensor:
    """Write rows [src_row, src_row + count) of each pair's CodeMatrix payload into records
    [dst_row, dst_row + count) of the group-major buffer gm [n_pairs, keycodes_gm_bytes(cap)] u8."""
    kd = _dev(kstack)
    if payload.dim() == 1:
        payload = payload.unsqueeze(0)
    stride = _pair_stride(payload, torch.uint8, "payload", 1)
    n_pairs = payload.shape[0]
    if gm is None:
        cap = cap or -(-max(count + dst_row, 1) // GM_ALIGN) * GM_ALIGN
        nb = keycodes_gm_bytes(kd, cap)
        if nb == 0:
            raise InvalidInput("stack has no group-major layout (D = 128, <= 1024 entries per stage)")
        gm = torch.zeros((n_pairs, nb), dtype=torch.uint8, device=payload.device)
    elif cap == 0:
        raise InvalidInput("cap is required with an existing group-major buffer")
    gstride = _pair_stride(gm, torch.uint8, "gm", 1)
    _lib.call("vqkv_keycodes_to_gm", kd.h, payload.data_ptr(), stride, n_pairs, src_row, count, gm.data_ptr(), cap,
              gstride, dst_row, _stream(payload))
    return gm


def keycodes_from_gm(kstack, gm: torch.Tensor, cap: int, count: int,
                     payload: Optional[torch.Tensor] = None) -> torch.Tensor:
    """CodeMatrix payloads [n_pairs, payload_bytes(count)] u8 of records [0, count) of the
    attention layout gm [n_pairs, keycodes_gm_bytes(cap)] (inverse of keycodes_to_gm)."""
    kd = _dev(kstack)
    if gm.dim() == 1:
        gm = gm.unsqueeze(0)
    gstride = _pair_stride(gm, torch.uint8, "gm", 1)
    n_pairs = gm.shape[0]
    pb = kd.payload_bytes(count)
    if payload is None:
        payload = torch.empty((n_pairs, max(pb, 1)), dtype=torch.uint8, device=gm.device)
    pstride = _pair_stride(payload, torch.uint8, "payload", 1)
    _lib.call("vqkv_keycodes_from_gm", kd.h, gm.data_ptr(), cap, gstride, n_pairs, count, payload.data_ptr(), pstride,
              _stream(gm))
    return payload


def attend_gm_supported(kstack, vstack, n_pairs: int, group: int, n_init: int, n_comp: int, n_local: int) -> bool:
    """Whether attend_decode takes group-major key codes for this shape (the LUT path covers it)."""
    import ctypes as C

    a = _lib.AttendArgs()
    a.n_pairs, a.group, a.n_init, a.n_comp, a.n_local = n_pairs, group, n_init, n_comp, n_local
    a.kcodes_layout = _lib.KEYCODES_GROUP_MAJOR
    return bool(_lib.load().vqkv_attend_gm_supported(_dev(kstack).h, _dev(vstack).h, C.byref(a)))


def attend_decode(
    kstack,
    vstack,
    q: torch.Tensor,
    kcodes: Optional[torch.Tensor],
    vcodes: Optional[torch.Tensor],
    n_comp: int,
    init_k: Optional[torch.Tensor] = None,
    init_v: Optional[torch.Tensor] = None,
    local_k: Optional[torch.Tensor] = None,
    local_v: Optional[torch.Tensor] = None,
    scale: float = 0.0,
    want_lse: bool = True,
    kcodes_gm_cap: int = 0,
) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """Decode-step attention for q [n_pairs, group, Dk] over init | compressed | local.

    init_k [n_pairs, n_init, Dk], local_k [n_pairs, n_local, Dk] (likewise V),
    kcodes/vcodes [n_pairs, payload_bytes(n_comp)] u8.  With kcodes_gm_cap > 0, kcodes is
    the group-major layout (keycodes_to_gm) with that capacity.  Returns (out [n_pairs, group, Dv],
    lse [n_pairs, group]).
    """
    kd, vd = _dev(kstack), _dev(vstack)
    _need(q, torch.float32, "q")
    n_pairs, group, dk = q.shape
    if dk != kd.dim:
        raise InvalidInput("query dimension does not match key dimension")
    n_init = 0 if init_k is None else init_k.shape[1]
    n_local = 0 if local_k is None else local_k.shape[1]
    strides = {}
    for t, nm in ((init_k, "init_k"), (init_v, "init_v"), (local_k, "local_k"), (local_v, "local_v"),
                  (kcodes if n_comp else None, "kcodes"), (vcodes if n_comp else None, "vcodes")):
        if t is not None:
            strides[nm] = _pair_stride(t, torch.uint8 if nm.endswith("codes") else torch.float32, nm, 1)
    # K and V segments share one stride each (same token layout)
    for a_, b_ in (("init_k", "init_v"), ("local_k", "local_v")):
        if strides.get(a_, 0) != strides.get(b_, 0):
            raise InvalidInput(f"{a_} and {b_} must have the same layout")
    out = torch.empty((n_pairs, group, vd.dim), dtype=torch.float32, device=q.device)
    lse = torch.empty((n_pairs, group), dtype=torch.float32, device=q.device) if want_lse else None
    a = _lib.AttendArgs(
        n_pairs, group, q.data_ptr(),
        init_k.data_ptr() if n_init else None, init_v.data_ptr() if n_init else None, n_init,
        kcodes.data_ptr() if n_comp else None, vcodes.data_ptr() if n_comp else None, n_comp,
        local_k.data_ptr() if n_local else None, local_v.data_ptr() if n_local else None, n_local,
        float(scale), out.data_ptr(), lse.data_ptr() if lse is not None else None,
        strides.get("init_k", 0), strides.get("local_k", 0), strides.get("kcodes", 0), strides.get("vcodes", 0),
        _lib.KEYCODES_GROUP_MAJOR if kcodes_gm_cap else _lib.KEYCODES_ROWS, kcodes_gm_cap,
    )
    import ctypes as C

    _lib.call("vqkv_attend_decode", kd.h, vd.h, C.byref(a), _stream(q))
    return out, lse


def lse_combine(parts_o: torch.Tensor, parts_lse: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """Merge sequence-split partials: parts_o [P, rows, dv], parts_lse [P, rows]."""
    _need(parts_o, torch.float32, "parts_o")
    _need(parts_lse, torch.float32, "parts_lse")
    P, rows, dv = parts_o.shape
    out = torch.empty((rows, dv), dtype=torch.float32, device=parts_o.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=parts_o.device)
    _lib.call("vqkv_lse_combine", parts_o.data_ptr(), parts_lse.data_ptr(), P, rows, dv, out.data_ptr(),
              lse.data_ptr(), _stream(parts_o))
    return out, lse


def set_encode_path(path: int) -> None:
    """0 auto, 1 exact SIMT, 2 tensor core (test hook)."""
    _lib.call("vqkv_set_encode_path", path)


def encode_counters(stack):
    import ctypes as C

    arr = (C.c_uint64 * 3)()
    _lib.call("vqkv_encode_counters", _dev(stack).h, arr)
    return dict(row_stages=arr[0], ambiguous=arr[1], exact_rows=arr[2])
