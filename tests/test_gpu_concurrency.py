"""The drop-in's concurrency and multi-process contracts on one B200.

* Two host threads with two different datasets at the same time give the same
  results as running alone (the reference's functions are pure and safe to
  call concurrently; its own depth_batch drives
  refined_random_search from a thread pool, optimizer.py:272-279).
* The product multi-GPU path (distributed.py) with the REAL engine
  (compute=None) under a world-size-2 process group whose ranks share cuda:0
  (gloo), bitwise equal to the single-process depth_batch_arrays: global query
  indices as Philox substreams, one all_gather.
* Queries outside the FP32 contraction range are rejected, like the dataset.
"""

import os
import socket
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_threads_two_datasets(b200):
    rng = np.random.default_rng(11)
    XA = rng.standard_normal((6000, 7))
    XB = rng.standard_normal((4100, 7)) * 3.0 + 1.0
    ZA, ZB = XA[:24], XB[:24] * 0.5
    cfgH = b200.RrsConfig(total_directions=2000, refinements=10, shrink=0.85, notion="halfspace", seed=5)
    cfgP = b200.RrsConfig(total_directions=800, refinements=8, shrink=0.85, notion="projection", seed=6)
    A, B = b200.Dataset(XA), b200.Dataset(XB)
    refA = b200.depth_batch_arrays(ZA, A, cfgH)
    refB = b200.depth_batch_arrays(ZB, B, cfgP)
    errors, results = [], {"A": [], "B": []}

    def worker(tag, Z, data, cfg):
        try:
            for _ in range(6):
                results[tag].append(b200.depth_batch_arrays(Z, data, cfg))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    ts = [threading.Thread(target=worker, args=("A", ZA, A, cfgH)),
          threading.Thread(target=worker, args=("B", ZB, B, cfgP))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for got in results["A"]:
        assert np.array_equal(got[0], refA[0]) and np.array_equal(got[1], refA[1])
    for got in results["B"]:
        assert np.array_equal(got[0], refB[0]) and np.array_equal(got[1], refB[1])


def _rank(rank, world, port, X, Z, out_path, device_path):
    import torch
    import torch.distributed as dist

    import paper_2506_08262_b200 as rrs
    from paper_2506_08262_b200.distributed import depth_sharded, depth_sharded_device, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both ranks on the one GPU of this box
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = rrs.RrsConfig(total_directions=1500, refinements=6, shrink=0.9, notion="halfspace", seed=3)
    data = rrs.Dataset(X)
    if device_path:
        eng = rrs.engine(0)
        eng.set_dataset(X, key="shard")
        a, b, S = shard_bounds(Z.shape[0], world, rank)
        Zs = np.zeros((S, X.shape[1]))
        Zs[: b - a] = Z[a:b]
        rec = depth_sharded_device(torch.from_numpy(Zs).cuda(), cfg, q_offset=a, eng=eng)
        torch.cuda.synchronize()
        rec = rec.cpu().numpy()
        # rows past this rank's slice are padding; keep each rank's real rows
        rows = np.concatenate([rec[g * S: g * S + (shard_bounds(Z.shape[0], world, g)[1] -
                                                    shard_bounds(Z.shape[0], world, g)[0])]
                               for g in range(world)])
        depth, cnt, argmin = rows[:, 0], rows[:, 1].astype(np.int64), rows[:, 2:]
    else:
        depth, cnt, argmin = depth_sharded(Z, data, cfg)
    if rank == 0:
        np.savez(out_path, depth=depth, cnt=cnt, argmin=argmin)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("device_path", [False, True])
def test_sharded_real_engine_two_ranks(b200, tmp_path, device_path):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(8)
    X = rng.standard_normal((5000, 9))
    Z = np.concatenate([X[:10], rng.standard_normal((5, 9))])  # Q = 15: uneven slices
    out = str(tmp_path / "res.npz")
    mp.spawn(_rank, args=(2, _free_port(), X, Z, out, device_path), nprocs=2, join=True)
    res = np.load(out)
    cfg = b200.RrsConfig(total_directions=1500, refinements=6, shrink=0.9, notion="halfspace", seed=3)
    depth, argmin, _, cnt = b200.depth_batch_arrays(Z, b200.Dataset(X), cfg)
    assert np.array_equal(res["depth"], depth)
    assert np.array_equal(res["argmin"], argmin)
    assert np.array_equal(res["cnt"], cnt)


def test_query_range_validation(b200):
    X = np.random.default_rng(1).standard_normal((300, 4))
    data = b200.Dataset(X)
    cfg = b200.RrsConfig(total_directions=100, refinements=2, notion="halfspace", seed=1)
    bad = [np.array([0.0, np.nan, 0.0, 0.0]), np.array([0.0, 0.0, np.inf, 0.0]),
           np.array([1e39, 0.0, 0.0, 0.0])]
    for z in bad:
        with pytest.raises(ValueError):
            b200.depth_batch_arrays(z[None, :], data, cfg)
        with pytest.raises(ValueError):
            b200.evaluate_directions(z, data, np.eye(4), "halfspace", b200.ParallelConfig())
    # the device-resident entry rejects them too
    import torch

    eng = b200.engine()
    eng.set_dataset(X, key="val")
    depth = torch.empty(1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        eng.depth_batch_device(torch.tensor([[0.0, np.nan, 0.0, 0.0]], device="cuda"), cfg, 0, depth)
    # a finite in-range query still works afterwards
    d, *_ = b200.depth_batch_arrays(X[:2], data, cfg)
    assert np.all(d > 0)
