"""The row-block pipeline driver (paper_1502_01645_b200/rowblock.py) across 3
ranks over gloo, with a CPU emulation of the chain continuation standing in
for the GPU kernels: the final Gram / A^T b / residual must be bitwise the
reference's (the C restatement's gram, transpose_matvec, residual)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1502_01645_b200.rowblock import chain_relay, pipelined_gram, row_split

D, N, SEED = 37, 9, 11
TILE = 7  # upper-triangle entries per emulated tile


def _problem():
    rng = np.random.default_rng(SEED)
    A = np.asfortranarray(rng.standard_normal((D, N)))
    b = rng.standard_normal(D)
    x = np.where(rng.uniform(size=N) < 0.5, 0.0, rng.uniform(size=N))
    return A, b, x


def _pairs():
    return [(i, j) for j in range(N) for i in range(j + 1)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, b, x = _problem()
    r0, r1 = row_split(D, world)[rank]
    pairs = _pairs()
    ntiles = (len(pairs) + TILE - 1) // TILE
    H = np.zeros((N, N))

    def compute(t0, t1, pin, pout):  # sequential chains over this block's rows
        for t in range(t0, t1):
            for e in range(TILE):
                idx = t * TILE + e
                if idx >= len(pairs):
                    continue
                i, j = pairs[idx]
                s = float(pin[(t - t0) * TILE + e]) if pin is not None else 0.0
                for k in range(r0, r1):
                    s = s + A[k, i] * A[k, j]
                if pout is not None:
                    pout[(t - t0) * TILE + e] = s
                else:
                    H[i, j] = H[j, i] = s

    pipelined_gram(dist, rank, world, ntiles, 2, TILE, compute, "cpu")

    def atb(pin):
        out = torch.zeros(N, dtype=torch.float64)
        for j in range(N):
            s = float(pin[j]) if pin is not None else 0.0
            for k in range(r0, r1):
                s = s + A[k, j] * b[k]
            out[j] = s
        return out

    h = chain_relay(dist, rank, world, torch.zeros(N, dtype=torch.float64), atb)

    def resid(pin):
        s = float(pin[0]) if pin is not None else 0.0
        for k in range(r0, r1):
            ax = 0.0
            for j in range(N):
                if x[j] != 0.0:
                    ax = ax + A[k, j] * x[j]
            r = ax - b[k]
            s = s + r * r
        return torch.tensor([s], dtype=torch.float64)

    rs = chain_relay(dist, rank, world, torch.zeros(1, dtype=torch.float64), resid)
    if rank == world - 1:
        np.savez(out_path, H=H, h=h.numpy(), r=rs.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_rowblock_pipeline_bitwise(tmp_path):
    from oracle.oracle import Oracle
    out = str(tmp_path / "rb.npz")
    mp.spawn(_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    got = np.load(out)
    A, b, x = _problem()
    o = Oracle("oracle")
    assert np.array_equal(got["H"].view(np.uint64), o.gram(A).view(np.uint64))
    assert np.array_equal(got["h"].view(np.uint64), o.transpose_matvec(A, b).view(np.uint64))
    ax = o.matvec(A, x)
    s = 0.0
    for k in range(D):
        r = ax[k] - b[k]
        s = s + r * r
    assert got["r"][0] == s


def test_row_split():
    assert row_split(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert row_split(32768, 8)[-1] == (28672, 32768)


# ---- configs[4] as written: partial Grams summed with one allreduce --------------------------
def _ar_worker(rank, world, port, out_path):
    from paper_1502_01645_b200.rowblock import allreduce_residual, allreduce_setup
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    A, b, x = _problem()
    r0, r1 = row_split(D, world)[rank]

    def compute(H, atb):  # this rank's partials (the GPU path: alnnls_gram_partial_device)
        Ab = A[r0:r1, :]
        H.copy_(torch.from_numpy(Ab.T @ Ab))
        atb.copy_(torch.from_numpy(Ab.T @ b[r0:r1]))

    H, atb = allreduce_setup(dist, world, N, compute, "cpu")
    r = A[r0:r1, :] @ x - b[r0:r1]
    res = allreduce_residual(dist, world, float(r @ r), "cpu")
    if rank == 0:
        np.savez(out_path, H=H.numpy(), h=atb.numpy(), r=np.array([res]))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_setup_two_ranks(tmp_path):
    out = str(tmp_path / "ar.npz")
    mp.spawn(_ar_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    A, b, x = _problem()
    assert np.allclose(got["H"], A.T @ A, rtol=1e-13, atol=1e-13)
    assert np.array_equal(got["H"], got["H"].T)
    assert np.allclose(got["h"], A.T @ b, rtol=1e-13, atol=1e-13)
    r = A @ x - b
    assert abs(got["r"][0] - float(r @ r)) <= 1e-12 * float(r @ r)
