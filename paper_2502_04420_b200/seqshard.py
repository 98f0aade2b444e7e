"""a6: sequence-sharded decode attention across GPUs.

Rank r of N holds tokens [start_r, end_r) of every (b, h) as a standalone cache.  Shard boundaries
are multiples of the KIVI flush size so every key block is identical to the unsharded cache's, and
only the last rank keeps a full-precision residual (the newest tokens live there, so appends go
there); the other ranks' specs use residual 0, i.e. every token they hold is quantised.  Per layer:

    partial (m, l, o) = kvt_decode_attention_partial(local cache)      [B][H_q][d + 2] fp32
    gathered = all_gather_into_tensor(partial)                          [N][B][H_q][d + 2]  (NCCL)
    out = kvt_combine_partials(gathered)                                 log-sum-exp merge (K3)

The exchange is the only collective of the whole path; it moves B·H_q·(d + 2)·4 bytes per rank per
layer (16.6 KB per sequence at Llama shape), so it is latency-bound.

`SymmExchange` fuses the exchange into the attention kernel instead: the gathered
buffer lives in symmetric memory, every rank's kernel stores its (m, l, o) rows straight into its slot of
every peer's buffer over NVLink (kvt_decode_attention_partial_push), one device-side barrier orders the
stores, and each rank combines its own buffer.  Two buffers alternate between layers, so one barrier per
layer suffices (a rank can only overwrite a peer's buffer k again after that peer passed the next barrier,
i.e. after its combine of buffer k).
"""
from __future__ import annotations

from dataclasses import replace
from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_bounds(total: int, world: int, rank: int, align: int = 32):
    """[start, end) of rank's token shard: equal shards rounded to `align` tokens, remainder on the last."""
    per = (total // world) // align * align
    start = rank * per
    end = total if rank == world - 1 else start + per
    return start, end


def shard_spec(spec, rank: int, world: int):
    """Non-final shards hold no residual: every token they own is quantised (residual 0)."""
    return spec if rank == world - 1 else replace(spec, residual=0)


def _all_gather(part: torch.Tensor, group=None, gathered: Optional[torch.Tensor] = None) -> torch.Tensor:
    if not dist.is_initialized():                          # one shard, no process group: nothing to exchange
        return part.unsqueeze(0)
    world = dist.get_world_size(group)
    if gathered is None:
        gathered = torch.empty((world,) + tuple(part.shape), dtype=part.dtype, device=part.device)
    try:
        dist.all_gather_into_tensor(gathered, part.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):
        dist.all_gather(list(gathered.unbind(0)), part.contiguous(), group=group)
    return gathered


def sharded_decode(cache, q: torch.Tensor, seq_len: torch.Tensor, seq_len_host=None, group=None,
                   out_dtype=torch.bfloat16, partial_fn: Optional[Callable] = None,
                   combine_fn: Optional[Callable] = None, scale: Optional[float] = None,
                   out: Optional[torch.Tensor] = None, part: Optional[torch.Tensor] = None,
                   gathered: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                   stream=None, after_partial: Optional[Callable] = None):
    """One layer of sequence-sharded decode attention on this rank; returns the full output on every rank.

    partial_fn / combine_fn default to the library's kernels; tests inject CPU stand-ins to exercise
    the orchestration (shard layout, gather order) on a gloo process group.  `part`, `gathered`, `out`
    and `workspace` are optional preallocated buffers (the benchmark's step reuses them every layer);
    `after_partial` is called right after the partial launch (the benchmark records a CUDA event there)."""
    if partial_fn is None:
        from . import kvt

        part = kvt.decode_attention_partial(cache, q, seq_len, seq_len_host=seq_len_host, scale=scale,
                                            partial=part, workspace=workspace, stream=stream)
    else:
        part = partial_fn(cache, q, seq_len)
    if after_partial is not None:
        after_partial()
    gathered = _all_gather(part, group, gathered)
    if combine_fn is None:
        from . import kvt

        return kvt.combine_partials(gathered, out=out, out_dtype=out_dtype, stream=stream)
    return combine_fn(gathered)


class SymmExchange:
    """Sequence-shard exchange over peer memory (no NCCL collective on the data path)."""

    def __init__(self, shape, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        full = (2, self.world) + tuple(shape)                  # [buffer][shard][B][H_q][d + 2]
        self.buf = symm_mem.empty(full, dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        peers = [self.handle.get_buffer(p, full, torch.float32) for p in range(self.world)]
        # slots[k][p] = this rank's slot of peer p's buffer k (a peer address mapped into this GPU)
        self.slots = [[peers[p][k, self.rank] for p in range(self.world)] for k in range(2)]
        self.k = 0

    def decode(self, cache, q, seq_len, seq_len_host=None, scale=None, out=None, out_dtype=torch.bfloat16,
               workspace=None, stream=None, after_partial: Optional[Callable] = None):
        from . import kvt

        k = self.k
        kvt.decode_attention_partial_push(cache, q, seq_len, self.slots[k], seq_len_host=seq_len_host, scale=scale,
                                          workspace=workspace, stream=stream)
        if after_partial is not None:
            after_partial()
        self.handle.barrier(channel=0)
        self.k ^= 1
        return kvt.combine_partials(self.buf[k], out=out, out_dtype=out_dtype, stream=stream)
