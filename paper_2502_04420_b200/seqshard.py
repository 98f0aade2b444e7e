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


def _all_gather(part: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    gathered = torch.empty((world,) + tuple(part.shape), dtype=part.dtype, device=part.device)
    try:
        dist.all_gather_into_tensor(gathered, part.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):
        dist.all_gather(list(gathered.unbind(0)), part.contiguous(), group=group)
    return gathered


def sharded_decode(cache, q: torch.Tensor, seq_len: torch.Tensor, seq_len_host=None, group=None,
                   out_dtype=torch.bfloat16, partial_fn: Optional[Callable] = None,
                   combine_fn: Optional[Callable] = None, scale: Optional[float] = None):
    """One layer of sequence-sharded decode attention on this rank; returns the full output on every rank.

    partial_fn / combine_fn default to the library's kernels; tests inject CPU stand-ins to exercise
    the orchestration (shard layout, gather order) on a gloo process group."""
    if partial_fn is None:
        from . import kvt

        part = kvt.decode_attention_partial(cache, q, seq_len, seq_len_host=seq_len_host, scale=scale)
    else:
        part = partial_fn(cache, q, seq_len)
    gathered = _all_gather(part, group)
    if combine_fn is None:
        from . import kvt

        return kvt.combine_partials(gathered, out_dtype=out_dtype)
    return combine_fn(gathered)
