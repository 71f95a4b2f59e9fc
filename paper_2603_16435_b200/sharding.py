"""Multi-GPU partitioning of the hot path.

* Encode / decode: the 256 (layer, KV-head) streams are independent
  (kv_cache.hpp:41-44) -> contiguous blocks of streams per
  rank, codebooks replicated, no collective.
* Decode attention, batch of sequences: shard KV heads (each rank owns the
  G query heads of its KV heads) -> no collective for the result.
* One long sequence: split the token range into contiguous shards -- raw
  init rows on shard 0, raw local window on the last shard, compressed rows
  split evenly -- each rank computes (o_r, lse_r); one exchange step
  (all-gather of o and lse over NCCL/NVLink) and every rank merges
      o = sum_r exp(lse_r - LSE) o_r,   LSE = log sum_r exp(lse_r).

Process model: one process per GPU under torchrun; torch.distributed is the
plumbing (NCCL on GPUs, gloo for the CPU tests).  The merge itself runs in
the library (vqkv_lse_combine) on GPUs; `lse_merge` is the same formula in
torch for CPU-side checks.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import torch


def stream_shard(n_streams: int, world: int, rank: int) -> range:
    """Contiguous block of (layer, head) streams owned by `rank` (balanced +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_streams, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def kv_head_shard(n_kv_heads: int, world: int, rank: int) -> range:
    """KV heads owned by `rank` for batched decode attention (G query heads each)."""
    return stream_shard(n_kv_heads, world, rank)


@dataclass(frozen=True)
class SeqShard:
    """Token ranges of one sequence shard, in the cache's token order."""

    init: Tuple[int, int]
    comp: Tuple[int, int]
    local: Tuple[int, int]

    @property
    def tokens(self) -> int:
        return sum(b - a for a, b in (self.init, self.comp, self.local))


def sequence_shards(n_init: int, n_comp: int, n_local: int, world: int) -> List[SeqShard]:
    """Split init | compressed | local over `world` ranks: init on rank 0, local on
    the last rank, compressed rows evenly (contiguous)."""
    out = []
    for r in range(world):
        c = stream_shard(n_comp, world, r)
        out.append(SeqShard(
            init=(0, n_init) if r == 0 else (0, 0),
            comp=(c.start, c.stop),
            local=(0, n_local) if r == world - 1 else (0, 0),
        ))
    return out


def lse_merge(o_parts: torch.Tensor, lse_parts: torch.Tensor) -> Tuple[torch.Tensor, torch.Tensor]:
    """o_parts [P, rows, dv], lse_parts [P, rows] -> (o [rows, dv], lse [rows]).

    Shards with no tokens carry lse = -inf and contribute nothing."""
    M = torch.max(lse_parts, dim=0).values
    w = torch.exp(lse_parts - M.unsqueeze(0))
    w = torch.where(torch.isfinite(lse_parts), w, torch.zeros_like(w))
    S = w.sum(0)
    o = (w.unsqueeze(-1) * o_parts).sum(0) / S.unsqueeze(-1)
    return o, M + torch.log(S)


def gather_and_merge(o_local: torch.Tensor, lse_local: torch.Tensor, group=None):
    """All-gather each rank's partial (o, lse) and merge identically on every rank.

    On CUDA tensors the exchange is one NCCL all-gather per tensor and the merge
    runs in the library's lse_combine kernel; on CPU (gloo) the torch formula."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    o_flat = o_local.contiguous().reshape(-1)
    l_flat = lse_local.contiguous().reshape(-1)
    o_all = torch.empty(world * o_flat.numel(), dtype=o_local.dtype, device=o_local.device)
    l_all = torch.empty(world * l_flat.numel(), dtype=lse_local.dtype, device=lse_local.device)
    dist.all_gather_into_tensor(o_all, o_flat, group=group)
    dist.all_gather_into_tensor(l_all, l_flat, group=group)
    rows = lse_local.numel()
    dv = o_local.shape[-1]
    if o_local.is_cuda:
        from . import device as Dv

        o, lse = Dv.lse_combine(o_all.reshape(world, rows, dv).contiguous(), l_all.reshape(world, rows).contiguous())
    else:
        o, lse = lse_merge(o_all.reshape(world, rows, dv), l_all.reshape(world, rows))
    return o.reshape(o_local.shape), lse.reshape(lse_local.shape)


class NcclComms:
    """ncclCommInitAll over local devices through the library (vqkv_nccl_comm_init_all): the
    single-process layout a C++ host uses for the 8-GPU sequence split."""

    def __init__(self, devices):
        import ctypes as C

        from . import _lib

        self.devices = list(devices)
        n = len(self.devices)
        self._h = (C.c_void_p * n)()
        _lib.call("vqkv_nccl_comm_init_all", n, (C.c_int * n)(*self.devices), self._h)

    def comm(self, i: int) -> int:
        return int(self._h[i])

    def close(self):
        from . import _lib

        for i in range(len(self.devices)):
            if self._h[i]:
                _lib.call("vqkv_nccl_comm_destroy", self._h[i])
                self._h[i] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_gather_and_merge(comm: int, o_local: torch.Tensor, lse_local: torch.Tensor):
    """The library's exchange step (vqkv_lse_allgather_combine): ncclAllGather of this rank's partial
    (o [rows, dv], lse [rows]) on the communicator's device, then the LSE merge -> (o, lse)."""
    from . import _lib

    if not (o_local.is_cuda and lse_local.is_cuda):
        raise ValueError("nccl_gather_and_merge needs CUDA tensors")
    o_local = o_local.contiguous()
    lse_local = lse_local.contiguous()
    rows = lse_local.numel()
    dv = o_local.shape[-1]
    out = torch.empty_like(o_local)
    out_lse = torch.empty_like(lse_local)
    s = torch.cuda.current_stream(o_local.device).cuda_stream
    _lib.call("vqkv_lse_allgather_combine", comm, o_local.data_ptr(), lse_local.data_ptr(), rows, dv, None, None,
              out.data_ptr(), out_lse.data_ptr(), s)
    return out, out_lse
