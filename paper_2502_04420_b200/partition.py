"""§8(e) work partition across GPUs (host logic only).

The decode path is independent per (sequence b, KV head h) unit: attention for query heads
h·g … h·g + g − 1 of sequence b reads only unit (b, h)'s cache ("sharing the same key cache" within a GQA
group; A10).  So a batch partitions across ranks with no data-path collective:

* B ≥ N — batch rows: rank r owns rows [⌊rB/N⌋, ⌊(r+1)B/N⌋) with all H KV heads (ragged when N ∤ B);
* B < N — KV heads: sequence b is owned by the ranks r with ⌊rB/N⌋ = b, which split its H KV heads into
  contiguous ranges (with their g query heads each).  Every (b, h) unit has exactly one owner.

Sequence sharding (config 5, a6) is the other partition (`seqshard.py`): every rank holds a token range
of every unit and one exchange per layer merges the partials.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Part:
    """Rank's share: batch rows [b_lo, b_hi) × KV heads [h_lo, h_hi) (query heads [h_lo·g, h_hi·g))."""
    b_lo: int
    b_hi: int
    h_lo: int
    h_hi: int

    @property
    def batch(self) -> int:
        return self.b_hi - self.b_lo

    @property
    def kv_heads(self) -> int:
        return self.h_hi - self.h_lo

    def units(self):
        return [(b, h) for b in range(self.b_lo, self.b_hi) for h in range(self.h_lo, self.h_hi)]


def partition(B: int, H: int, world: int, rank: int) -> Part:
    if not (B >= 1 and H >= 1 and world >= 1 and 0 <= rank < world):
        raise ValueError(f"bad partition arguments B={B} H={H} world={world} rank={rank}")
    if B >= world:
        return Part(rank * B // world, (rank + 1) * B // world, 0, H)
    if B * H < world:
        raise ValueError(f"{B} sequences x {H} KV heads cannot give each of {world} ranks a unit")
    b = rank * B // world
    owners = [r for r in range(world) if r * B // world == b]          # contiguous ranks sharing sequence b
    k, i = len(owners), rank - owners[0]
    return Part(b, b + 1, i * H // k, (i + 1) * H // k)


def strong_scaling_plan(global_batch: int, H: int, world: int):
    """Every rank's Part for a fixed global batch (strong scaling)."""
    return [partition(global_batch, H, world, r) for r in range(world)]
