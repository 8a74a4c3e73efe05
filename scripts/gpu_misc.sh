cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "layout_dims" > gpurun_out/layout_tests.log 2>&1; echo "rc=$?" >> gpurun_out/layout_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 1 --batch 256 --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 > gpurun_out/bench_ref_torchrun1.json 2> gpurun_out/bench_ref_torchrun1.err
cat > /tmp/c5.py <<'PY'
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2506_08262_b200 as rrs
from paper_2506_08262_b200.synthetic import toeplitz_gaussian
X = toeplitz_gaussian(200, 1_000_000, seed=0)
data = rrs.Dataset(X)
for notion, q, k, r in (("halfspace", 8, 20000, 20), ("projection", 2, 2000, 20)):
    cfg = rrs.RrsConfig(total_directions=k, refinements=r, shrink=0.9, notion=notion, seed=1)
    t0 = time.time(); out = rrs.depth_batch_arrays(X[:q], data, cfg); dt = time.time() - t0
    print(notion, "queries", q, "k", k, "r", r, "time", round(dt, 2), "s ->", round(q / dt, 3), "q/s; depths", out[0][:4], flush=True)
PY
timeout 900 python /tmp/c5.py > gpurun_out/config5.log 2>&1; echo "rc=$?" >> gpurun_out/config5.log
echo done
