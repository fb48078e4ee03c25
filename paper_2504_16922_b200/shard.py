"""Host-side sharding of the GNA forward across ranks (one process per GPU).

The path has no exchange step: (batch, head) units are independent, and inside
one (batch, head) the work items (Q sub-tile pairs) are independent too.
  * weak scaling  -- each rank owns whole units of a global batch (unit_range);
  * Q-tile split  -- one problem's global work list [0, n_work) is cut into
    contiguous balanced ranges (work_range) handed to gna_forward_ex /
    gna_attention_permuted as [work_begin, work_end).
No collective touches the data path; verification gathers are separate.
"""
from __future__ import annotations


def balanced_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of rank's contiguous share; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def unit_range(batch: int, heads: int, world: int, rank: int) -> tuple[int, int]:
    """Units u = b*heads + h owned by rank (weak/strong batch x heads split)."""
    return balanced_range(batch * heads, world, rank)


def work_range(n_work: int, world: int, rank: int) -> tuple[int, int]:
    """Q-tile split of one problem's global work list."""
    return balanced_range(n_work, world, rank)
