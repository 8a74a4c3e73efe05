cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "large_rows" > gpurun_out/large_tests.log 2>&1; echo "rc=$?" >> gpurun_out/large_tests.log
cat > /tmp/c5p.py <<'PY'
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2506_08262_b200 as rrs
from paper_2506_08262_b200.synthetic import toeplitz_gaussian
X = toeplitz_gaussian(200, 1_000_000, seed=0)
data = rrs.Dataset(X)
eng = rrs.engine(); eng.enable_timing(True)
cfg = rrs.RrsConfig(total_directions=2000, refinements=20, shrink=0.9, notion="projection", seed=1)
rrs.depth_batch_arrays(X[:1], data, cfg)
t0 = time.time(); out = rrs.depth_batch_arrays(X[:2], data, cfg); dt = time.time() - t0
print("projection n=1M d=200 2 queries k=2000:", round(dt, 3), "s", out[0], eng.stats(), flush=True)
PY
timeout 600 python /tmp/c5p.py > gpurun_out/c5p.log 2>&1; echo "rc=$?" >> gpurun_out/c5p.log
echo done
