"""Query sharding over one process per GPU.

Each query's RRS is independent (only the pole chain inside a query is
sequential, optimizer.py:174), so the path shards with no data-path
collective: rank g owns the contiguous slice [g*S, (g+1)*S) of the query list
(S = ceil(Q / world)), the dataset is replicated on every GPU, and every query
keeps its GLOBAL index as its Philox substream (optimizer.py:254-279), so the
result is bitwise independent of the world size.  The single collective is one
all_gather of fixed-stride per-query records at the end:

    record = [depth, min_count, argmin[0..d)]   (float64, 2 + d words)

Over NCCL (backend "nccl") that is one ncclAllGather on NVLink; the same code
runs under gloo on CPU for the host-side tests, with the per-rank compute
injected (the oracle), since there is no CPU path in the product.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(Q: int, world: int, rank: int) -> tuple[int, int, int]:
    """(start, stop, padded slice size) of `rank`'s contiguous query slice."""
    S = -(-Q // world) if Q else 0
    start = min(rank * S, Q)
    stop = min(start + S, Q)
    return start, stop, S


def pack_records(depth, count, argmin, S: int) -> np.ndarray:
    d = argmin.shape[1] if argmin.ndim == 2 else 0
    rec = np.zeros((S, 2 + d))
    k = depth.shape[0]
    rec[:k, 0] = depth
    rec[:k, 1] = count
    if d:
        rec[:k, 2:] = argmin
    return rec


def unpack_records(all_rec: np.ndarray, Q: int):
    all_rec = all_rec[:Q]
    return all_rec[:, 0].copy(), all_rec[:, 1].astype(np.int64), all_rec[:, 2:].copy()


def depth_sharded(queries, data, cfg, *, group=None, compute=None, device=None):
    """Sharded depth_batch over torch.distributed.  Returns (depth, min_count,
    argmin) for ALL queries on every rank.

    compute(Z_slice, q0) -> (depth, count, argmin) overrides the per-rank
    solver (tests inject the CPU oracle under gloo; the product uses the B200
    engine)."""
    import torch
    import torch.distributed as dist

    Z = np.ascontiguousarray(queries, dtype=np.float64)
    Q, d = Z.shape
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, stop, S = shard_bounds(Q, world, rank)
    if compute is None:
        from .solver import depth_batch_arrays

        def compute(Zs, q0):
            if Zs.shape[0] == 0:
                return np.empty(0), np.empty(0, dtype=np.int64), np.empty((0, d))
            depth, argmin, _, cnt = depth_batch_arrays(Zs, data, cfg, q0=q0, device=device)
            return depth, cnt, argmin

    depth, count, argmin = compute(Z[start:stop], start)
    rec = pack_records(np.asarray(depth), np.asarray(count), np.asarray(argmin).reshape(-1, d), S)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    local = torch.from_numpy(rec).to(dev)
    gathered = torch.empty((world * S, 2 + d), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(gathered, local, group=group)
    return unpack_records(gathered.cpu().numpy(), Q)


def depth_sharded_device(Z_dev, cfg, *, q_offset: int, eng, group=None):
    """Device-resident variant for the benchmark: Z_dev is this rank's CUDA
    float64 slice (S, d); returns the gathered CUDA record tensor (world*S, 2+d)
    after ONE all_gather_into_tensor (NCCL over NVLink)."""
    import torch
    import torch.distributed as dist

    S, d = Z_dev.shape
    rec = torch.empty((S, 2 + d), dtype=torch.float64, device=Z_dev.device)
    depth = torch.empty(S, dtype=torch.float64, device=Z_dev.device)
    argmin = torch.empty((S, d), dtype=torch.float64, device=Z_dev.device)
    count = torch.empty(S, dtype=torch.int64, device=Z_dev.device)
    # the engine launches on its own stream unless bound to torch's: bind it to the
    # current torch stream so the reads below are stream-ordered after the kernels
    # (torch's legacy default stream has handle 0, which the ABI reads as "own
    # stream", so that case synchronises instead)
    cur = torch.cuda.current_stream(Z_dev.device)
    with eng.lock:
        if cur.cuda_stream:
            eng.set_stream(cur.cuda_stream)
        eng.depth_batch_device(Z_dev, cfg, q_offset, depth, argmin, None, count, eps=cfg.epsilons())
        if not cur.cuda_stream:
            eng.synchronize()
    rec[:, 0] = depth
    rec[:, 1] = count.to(torch.float64)
    rec[:, 2:] = argmin
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return rec
    if dist.get_backend(group) != "nccl":
        # gloo (ranks sharing one GPU in the single-GPU rehearsal): the same one
        # all_gather, staged through host memory
        host = rec.cpu()
        gathered = torch.empty((world * S, 2 + d), dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, host, group=group)
        return gathered.to(Z_dev.device)
    gathered = torch.empty((world * S, 2 + d), dtype=torch.float64, device=Z_dev.device)
    dist.all_gather_into_tensor(gathered, rec, group=group)
    return gathered
