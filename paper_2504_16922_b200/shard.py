"""Host-side partition of one GNA forward across ranks (one process per GPU).

The path has no exchange step (BASELINE.json north_star): the units
u = b*heads + h are independent, and inside one unit the work items (Q sub-tile pairs)
are independent too.  A problem of B x H units is split over G ranks as

  * "heads"  -- H >= G: rank r owns heads [h0, h1) of every sample (balanced), held as its
                own contiguous [B, *spatial, h1-h0, D] shard;
  * "batch"  -- otherwise, B >= G: rank r owns samples [b0, b1) (balanced), shard
                [b1-b0, *spatial, H, D];
  * "qtile"  -- fewer units than ranks (single-sample video with few heads): every rank
                holds the whole (replicated) problem and runs a contiguous balanced range
                [w0, w1) of the global work list (n_work = B*H*n_items, unit-major) through
                gna_forward_ex's work range -- Q-tile splitting.

No collective touches the data path; the verification gather is separate and untimed.
"""
from __future__ import annotations

import dataclasses


def balanced_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of rank's contiguous share; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def unit_range(batch: int, heads: int, world: int, rank: int) -> tuple[int, int]:
    """Units u = b*heads + h owned by rank (contiguous balanced split of B x H)."""
    return balanced_range(batch * heads, world, rank)


def work_range(n_work: int, world: int, rank: int) -> tuple[int, int]:
    """Q-tile split of one problem's global work list."""
    return balanced_range(n_work, world, rank)


@dataclasses.dataclass(frozen=True)
class Shard:
    mode: str                 # "heads" | "batch" | "qtile"
    rank: int
    world: int
    batch: tuple              # [b0, b1) of the global batch held by this rank
    heads: tuple              # [h0, h1) of the global heads held by this rank
    work: tuple | None        # qtile: [w0, w1) of the global work list, else None

    @property
    def shard_batch(self) -> int:
        return self.batch[1] - self.batch[0]

    @property
    def shard_heads(self) -> int:
        return self.heads[1] - self.heads[0]

    def units(self, heads_total: int) -> list[int]:
        """Global units u = b*H + h this rank computes completely (qtile: partially)."""
        return [b * heads_total + h for b in range(*self.batch) for h in range(*self.heads)]


def partition(batch: int, heads: int, world: int, rank: int, n_items: int, mode: str = "auto") -> Shard:
    """The shard of `rank` (see module doc).  mode: auto | heads | batch | qtile."""
    if mode == "auto":
        mode = "heads" if heads >= world else ("batch" if batch >= world else "qtile")
    if mode == "heads":
        if heads < world:
            raise ValueError(f"heads partition needs heads >= world ({heads} < {world})")
        return Shard("heads", rank, world, (0, batch), balanced_range(heads, world, rank), None)
    if mode == "batch":
        if batch < world:
            raise ValueError(f"batch partition needs batch >= world ({batch} < {world})")
        return Shard("batch", rank, world, balanced_range(batch, world, rank), (0, heads), None)
    if mode == "qtile":
        return Shard("qtile", rank, world, (0, batch), (0, heads),
                     work_range(batch * heads * n_items, world, rank))
    raise ValueError(f"unknown partition mode {mode!r}")
