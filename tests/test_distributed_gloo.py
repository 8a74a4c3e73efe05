"""Query sharding (world size 2, gloo, CPU): global query indices, padding,
one all_gather of fixed-stride records; the per-rank solver is the CPU oracle
(injected), so the host logic is exercised without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_08262_b200.distributed import pack_records, shard_bounds, unpack_records


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_bounds_cover_everything():
    for Q in (0, 1, 7, 8, 1001):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                a, b, S = shard_bounds(Q, world, r)
                assert b - a <= S
                seen.extend(range(a, b))
            assert seen == list(range(Q))


def test_pack_unpack_roundtrip():
    depth = np.array([0.1, 0.2, 0.3])
    cnt = np.array([1, 2, 3])
    argmin = np.arange(6.0).reshape(3, 2)
    rec = pack_records(depth, cnt, argmin, 4)
    assert rec.shape == (4, 4)
    d, c, a = unpack_records(rec, 3)
    assert np.array_equal(d, depth) and np.array_equal(c, cnt) and np.array_equal(a, argmin)


def _worker(rank, world, port, X, Z, out_path):
    import torch.distributed as dist

    from oracle import oracle
    from paper_2506_08262_b200.config import Dataset, RrsConfig
    from paper_2506_08262_b200.distributed import depth_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = RrsConfig(total_directions=300, refinements=6, shrink=0.9, notion="halfspace", seed=3)

    def compute(Zs, q0):
        depth, argmin, _ = oracle.depth_batch(Zs, X, total_directions=300, refinements=6, shrink=0.9,
                                              notion="halfspace", seed=3, q0=q0, threads=1)
        return depth, np.rint(depth * X.shape[0]), argmin

    depth, cnt, argmin = depth_sharded(Z, Dataset(X), cfg, compute=compute)
    if rank == 0:
        np.savez(out_path, depth=depth, cnt=cnt, argmin=argmin)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("Q", [13, 16])
def test_sharded_equals_single_process(tmp_path, orc, Q):
    rng = np.random.default_rng(5)
    X = rng.standard_normal((150, 4))
    Z = np.concatenate([X[:Q - 3], rng.standard_normal((3, 4))])
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), X, Z, out), nprocs=2, join=True)
    res = np.load(out)
    depth, argmin, _ = orc.depth_batch(Z, X, total_directions=300, refinements=6, shrink=0.9,
                                       notion="halfspace", seed=3)
    assert np.array_equal(res["depth"], depth)
    assert np.array_equal(res["argmin"], argmin)
    assert np.array_equal(res["cnt"], np.rint(depth * 150).astype(np.int64))
