"""Column sharding of a batched multi-RHS solve across ranks (BASELINE.json c4:
"independent right-hand sides ... split by column across 1/2/4/8 GPUs with no
communication"). Every column is an independent solve_nnls(A, B[:, j], cfg)
(reference nnls.hpp:129-144), so a rank owns a contiguous column range and no
data-path collective exists; only the timing reduction (max over ranks) and an
optional result gather cross ranks.
"""


def column_shard(ncols, world, rank):
    """Balanced contiguous split: returns (first column, count) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_shard: bad world/rank")
    base, extra = divmod(ncols, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_columns(dist, local, ncols, world, rank):
    """Assembles the (rows x ncols) result on every rank from per-rank column
    blocks (torch tensors, column-major stored as (count, rows) row-major)."""
    import torch
    counts = [column_shard(ncols, world, r)[1] for r in range(world)]
    rows = local.shape[1]
    width = max(counts)
    buf = torch.zeros((width, rows), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return torch.cat([o[:c] for o, c in zip(out, counts)], dim=0)
