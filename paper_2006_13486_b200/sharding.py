"""Batch / column sharding of the RBGP4 product across GPUs (one process per GPU).

Output columns are independent: tile (tbm, tbn) of O depends only on the
columns tbn*tn..(tbn+1)*tn of I (reference `sdmm.py:167-175`).  So each rank
multiplies the replicated W against its own contiguous slice of the columns
of I -- no communication on the hot path ("scaling: weak" when every rank
brings its own batch).  `gather_columns` is the single collective, an
all-gather of the column shards used only to assemble O for verification;
over NCCL it runs on NVLink/NVSwitch, under gloo it runs on the CPU (tests).

Shard boundaries are multiples of `tn` so every rank still satisfies the
reference's `N % tn == 0` contract on its own slice (the last rank takes any
remainder tiles when tiles do not divide evenly).
"""

from __future__ import annotations

from .errors import ConfigurationError


def column_shards(n_cols: int, world_size: int, tn: int = 1):
    """Contiguous [start, stop) column ranges, one per rank, tile-aligned."""
    if world_size < 1:
        raise ConfigurationError([f"world_size must be positive, got {world_size}"])
    if tn < 1 or n_cols % tn:
        raise ConfigurationError([f"input columns {n_cols} not divisible by tn={tn}"])
    tiles = n_cols // tn
    base, extra = divmod(tiles, world_size)
    out, start = [], 0
    for r in range(world_size):
        count = base + (1 if r < extra else 0)
        out.append((start * tn, (start + count) * tn))
        start += count
    return out


def shard_of(n_cols: int, world_size: int, rank: int, tn: int = 1):
    return column_shards(n_cols, world_size, tn)[rank]


def local_columns(inp, world_size: int, rank: int, tn: int = 1):
    """This rank's column slice of a replicated I (a view, no copy)."""
    start, stop = shard_of(inp.shape[1], world_size, rank, tn)
    return inp[:, start:stop]


def rbgp4mm_sharded(w, inp_local, params, *, compute: str = "exact", multiply=None):
    """O_local = W x I_local on this rank's GPU; no collective involved.

    `inp_local` is this rank's column shard (see `local_columns`).  `multiply`
    defaults to the CUDA product `rbgp4mm`; it is a parameter only so the
    host-side sharding logic can be exercised by CPU tests.
    """
    if multiply is None:
        from .sdmm import rbgp4mm as multiply
        return multiply(w, inp_local, params, compute=compute)
    return multiply(w, inp_local, params)


def gather_columns(local_out, n_cols: int, tn: int = 1, group=None):
    """Assemble the full (rows, n_cols) O from every rank's column shard.

    Verification only (never on the hot path): pads each shard to the widest
    one, all-gathers, and concatenates along columns in rank order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    shards = column_shards(n_cols, world, tn)
    width = max(b - a for a, b in shards)
    rows = local_out.shape[0]
    padded = local_out.new_zeros((rows, width))
    padded[:, : local_out.shape[1]] = local_out
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded.contiguous(), group=group)
    return torch.cat([buf[:, : b - a] for buf, (a, b) in zip(bufs, shards)], dim=1)
