"""Multi-rank column sharding of the batched (c4) path on CPU: world_size 2 over
gloo. Each rank solves its column shard with the CPU restatement (the checker,
standing in for the per-rank GPU solve), the shards are gathered, and the
result must be bitwise the unsharded per-column solve (no cross-rank data
exchange exists on the path, so sharding cannot change any bit)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1502_01645_b200.sharding import column_shard, gather_columns


def test_column_shard_covers_exactly():
    for ncols in (0, 1, 7, 64, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s, c = column_shard(ncols, world, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(ncols))
            counts = [column_shard(ncols, world, r)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        column_shard(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_1502_01645_b200 import instances
    from paper_1502_01645_b200.api import SolverConfig
    ncols = 9
    inst = instances.make_batched(d=90, n=24, nrhs=ncols, seed=5)
    col0, cnt = column_shard(ncols, world, rank)
    o = Oracle("oracle")
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9).to_abi()
    local = torch.zeros((cnt, inst["A"].shape[1]), dtype=torch.float64)
    iters = torch.zeros(ncols, dtype=torch.int64)
    for k in range(cnt):
        r = o.solve_nnls(inst["A"], inst["B"][:, col0 + k].copy(), cfg)
        local[k] = torch.from_numpy(np.asarray(r["x"]))
        iters[col0 + k] = int(r["iterations"])
    X = gather_columns(dist, local, ncols, world, rank)
    dist.all_reduce(iters)  # disjoint shards: the sum is the concatenation
    if rank == 0:
        np.savez(out_path, X=X.numpy(), iters=iters.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_batched_equals_unsharded(tmp_path):
    from oracle.oracle import Oracle
    from paper_1502_01645_b200 import instances
    from paper_1502_01645_b200.api import SolverConfig
    out = str(tmp_path / "sharded.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    inst = instances.make_batched(d=90, n=24, nrhs=9, seed=5)
    o = Oracle("oracle")
    cfg = SolverConfig(epsilon=1e-8, stall_window=10**9).to_abi()
    for j in range(9):
        r = o.solve_nnls(inst["A"], inst["B"][:, j].copy(), cfg)
        assert np.array_equal(got["X"][j].view(np.uint64), np.asarray(r["x"]).view(np.uint64)), j
        assert got["iters"][j] == r["iterations"]
