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


def _pack_torch(H, P):
    n = H.shape[0]
    tri = torch.triu_indices(n, n, device=H.device)
    P.copy_(H[tri[0], tri[1]])


def _unpack_torch(P, H):
    n = H.shape[0]
    tri = torch.triu_indices(n, n, device=H.device)
    H[tri[0], tri[1]] = P
    H[tri[1], tri[0]] = P


def allreduce_setup(dist, world, n, compute, device, pack=None, unpack=None):
    """BASELINE.json configs[4] as written (SURVEY.md §8e variant (i)): every rank
    forms the partial Gram of its row block and its partial A^T b, and the
    partials are summed with ONE allreduce (NCCL over NVLink between GPUs, gloo
    in the CPU tests). The collective moves the packed upper triangle of H and
    A^T b in one buffer: n(n+1)/2 + n doubles (1.07 GB at c5 instead of 2.15 GB
    for both triangles; H is exactly symmetric, so the lower half is mirrored
    back afterwards).

    compute(H, atb) fills this rank's partials in place (H: n x n, both
    triangles; atb: a view into the collective's buffer). pack(H, P) / unpack(P,
    H) convert to and from the packed layout (the GPU path passes the C ABI's
    alnnls_pack_upper_device / alnnls_unpack_upper_device; the default uses
    torch indexing, for small CPU tests). Returns the summed (H, atb) on every
    rank. The cross-rank sum order is the collective's, so H equals the
    reference's gram only within rounding; the pipelined_gram path is the
    bitwise one."""
    npk = n * (n + 1) // 2
    H = torch.empty((n, n), dtype=torch.float64, device=device)
    buf = torch.empty(npk + n, dtype=torch.float64, device=device)
    atb = buf[npk:]
    compute(H, atb)
    (pack or _pack_torch)(H, buf[:npk])
    if dist is not None and world > 1:
        dist.all_reduce(buf)
    (unpack or _unpack_torch)(buf[:npk], H)
    return H, atb


def allreduce_residual(dist, world, partial, device):
    """residual_norm_sq (nnls.hpp:115-123) as the sum of the ranks' row-block
    partial chains (one allreduce of one scalar)."""
    t = torch.tensor([float(partial)], dtype=torch.float64, device=device)
    if dist is not None and world > 1:
        dist.all_reduce(t)
    return float(t[0])
