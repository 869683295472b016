"""Exact multi-GPU setup by row blocks (BASELINE.json c5; SURVEY.md §8e variant (ii)).

A (d x n) is split into contiguous row blocks, one per rank. Every sum of the
reference setup is ONE ascending chain over the rows of A (gram linalg.hpp:168,
transpose_matvec linalg.hpp:215, residual_norm_sq nnls.hpp:119-122), so rank p
continues the chain states rank p-1 handed it and passes its own on: the last
rank ends with the reference's Gram bit for bit. The Gram states travel per
batch of output tiles, so after a (world - 1)-batch fill every rank computes a
different batch concurrently (a pipeline), and each batch crosses each link once.

The driver is backend-agnostic: `compute_*` callbacks do the arithmetic (the
GPU path calls the C ABI's *_rowblock_device entries; tests use a CPU
emulation) and `torch.distributed` moves the states (NCCL between GPUs, gloo in
the CPU tests).
"""
import torch


def row_split(d, world):
    """Balanced contiguous row blocks: [(r0, r1)] per rank."""
    base, extra = divmod(d, world)
    out, r = [], 0
    for p in range(world):
        c = base + (1 if p < extra else 0)
        out.append((r, r + c))
        r += c
    return out


def _finish_send(work, device):
    """Blocks the HOST until an isend has completed. With NCCL, Work.wait() only
    makes torch's current stream wait for the collective stream; the compute
    callbacks write their output buffers on the library's own stream, which is
    not ordered after that wait, so reusing a send buffer needs the host to see
    the send finish first (gloo's wait() already blocks the host)."""
    work.wait()
    if torch.device(device).type == "cuda":
        torch.cuda.current_stream(torch.device(device)).synchronize()


def pipelined_gram(dist, rank, world, ntiles, batch, tile_doubles, compute, device,
                   sync=None):
    """Runs the row-block Gram pipeline over `ntiles` tiles in batches.

    compute(t0, t1, pin, pout): continue tiles [t0, t1) of this rank's block from
    the states `pin` (None on rank 0) into `pout` (None on the last rank, which
    finishes the Gram). pin/pout are 1-D float64 tensors of (t1-t0)*tile_doubles.
    `sync()` makes received data visible to the compute engine (GPU: a stream
    synchronize; the callbacks return after their work is done).
    """
    nb = (ntiles + batch - 1) // batch
    cap = batch * tile_doubles
    first, last = rank == 0, rank == world - 1
    bin_ = [torch.empty(cap, dtype=torch.float64, device=device) for _ in range(2)] if not first else None
    bout = [torch.empty(cap, dtype=torch.float64, device=device) for _ in range(2)] if not last else None
    sends = [None] * nb

    def span(b):
        t0 = b * batch
        t1 = min(ntiles, t0 + batch)
        return t0, t1, (t1 - t0) * tile_doubles

    recv = None
    if not first and nb > 0:
        recv = dist.irecv(bin_[0][: span(0)[2]], src=rank - 1)
    for b in range(nb):
        t0, t1, cnt = span(b)
        pin = None
        if not first:
            recv.wait()
            if sync:
                sync()
            pin = bin_[b % 2][:cnt]
            if b + 1 < nb:  # the other buffer held batch b-1, already consumed
                recv = dist.irecv(bin_[(b + 1) % 2][: span(b + 1)[2]], src=rank - 1)
        if last:
            compute(t0, t1, pin, None)
        else:
            if b >= 2 and sends[b - 2] is not None:
                _finish_send(sends[b - 2], device)  # bout[b % 2] is free again
                sends[b - 2] = None
            pout = bout[b % 2][:cnt]
            compute(t0, t1, pin, pout)
            sends[b] = dist.isend(pout, dst=rank + 1)
    for w in sends:
        if w is not None:
            _finish_send(w, device)


def chain_relay(dist, rank, world, state, compute, sync=None):
    """Sequential relay of a chain state (a 1-D tensor) through the ranks in
    order: rank p receives the state of ranks < p, continues it with
    compute(state_in or None) -> state_out, and sends it on. Returns the final
    state on the last rank (None elsewhere)."""
    pin = None
    if rank > 0:
        pin = torch.empty_like(state)
        dist.recv(pin, src=rank - 1)
        if sync:
            sync()
    out = compute(pin)
    if rank < world - 1:
        dist.send(out, dst=rank + 1)
        return None
    return out


def allreduce_setup(dist, world, n, compute, device):
    """BASELINE.json configs[4] as written (SURVEY.md §8e variant (i)): every rank
    forms the partial Gram of its row block and its partial A^T b, and the
    partials are summed with ONE allreduce (NCCL over NVLink between GPUs, gloo
    in the CPU tests). H and A^T b share one buffer so the single collective
    moves both: n*n + n doubles (H is symmetric, so its n x n view is the same
    in either storage order).

    compute(H, atb) fills this rank's partials in place. Returns the summed
    (H, atb) on every rank. The cross-rank sum order is the collective's, so H
    equals the reference's gram only within rounding; the pipelined_gram path
    is the bitwise one."""
    buf = torch.empty(n * n + n, dtype=torch.float64, device=device)
    H = buf[: n * n].view(n, n)
    atb = buf[n * n:]
    compute(H, atb)
    if dist is not None and world > 1:
        dist.all_reduce(buf)
    return H, atb


def allreduce_residual(dist, world, partial, device):
    """residual_norm_sq (nnls.hpp:115-123) as the sum of the ranks' row-block
    partial chains (one allreduce of one scalar)."""
    t = torch.tensor([float(partial)], dtype=torch.float64, device=device)
    if dist is not None and world > 1:
        dist.all_reduce(t)
    return float(t[0])
