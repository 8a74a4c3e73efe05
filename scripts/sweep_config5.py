"""BASELINE config 5 sweep on one B200: halfspace + projection depth RRS,
n = 1M, d = 200 (Toeplitz Gaussian), k = 20,000, r in {10, 20, 40} x
sphcap_shrink alpha in {0.6, 0.7, 0.8, 0.9} († values).

Every cell runs the same FIXED query subset: contiguous rows from an offset
drawn by np.random.Philox(key=3) (rows are i.i.d.; SURVEY §8(d) asks for a
fixed random subset), with global query indices = row indices, so cells are
comparable: W warm-up batches, then K timed batches bracketed by CUDA events on
the engine stream, L2 flushed between batches, nvidia-smi clocks sampled over
the timed region (bench.py's ClockSampler).  One dataset upload per notion.

    python scripts/sweep_config5.py --out profiles/r2/config5_sweep.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_08262_b200 as rrs  # noqa: E402
from paper_2506_08262_b200.distributed import depth_sharded_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "config5_sweep.json"))
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=200)
ap.add_argument("--notions", default="halfspace,projection")
args = ap.parse_args()

n, d, k = args.n, args.d, 20_000
BATCH = {"halfspace": 16, "projection": 4}
X = bench.make_data("gaussian", n, d)
s0 = int(np.random.Generator(np.random.Philox(key=3)).integers(0, n - 8192))  # the fixed query subset
eng = rrs.engine(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.set_stream(stream.cuda_stream)
eng.set_dataset(X, key="sweep")
Xd = torch.from_numpy(X).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for notion in args.notions.split(","):
    B = BATCH[notion]
    for r in (10, 20, 40):
        for alpha in (0.6, 0.7, 0.8, 0.9):
            cfg = rrs.RrsConfig(total_directions=k, refinements=r, shrink=alpha, notion=notion, seed=1)
            batches = [(s0 + s * B, Xd[s0 + s * B:s0 + (s + 1) * B].contiguous())
                       for s in range(args.warmup + args.steps)]
            depths = []

            def run(q0, Z):
                return depth_sharded_device(Z, cfg, q_offset=q0, eng=eng)[:, 0]

            for s in range(args.warmup):
                run(*batches[s])
            torch.cuda.synchronize()
            clocks = bench.ClockSampler(0)
            clocks.start()
            ms = 0.0
            for s in range(args.warmup, args.warmup + args.steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                dep = run(*batches[s])
                b.record(stream)
                torch.cuda.synchronize()
                ms += a.elapsed_time(b)
                depths.append(dep.cpu().numpy())
            clk = clocks.stop()
            q = args.steps * B
            row = {"notion": notion, "r": r, "alpha": alpha, "m": -(-k // r), "queries_timed": q,
                   "ms": ms, "query_depths_per_s": q / (ms / 1e3),
                   "mean_depth": float(np.mean(np.concatenate(depths))), "clocks": clk}
            rows.append(row)
            print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as fh:
    json.dump({"workload": "BASELINE config 5: n=1M, d=200 Gaussian, k=20000, r x alpha sweep, fixed query "
                           "subset (contiguous rows from a np.random.Philox(key=3) offset), one B200",
               "generated": time.strftime("%Y-%m-%d %H:%M:%S"), "cells": rows}, fh, indent=1)
print("wrote", args.out)
