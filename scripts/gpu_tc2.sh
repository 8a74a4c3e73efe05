# first run of the 2-SM kernel: tiny shape under a short timeout, then parity, then bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/t2.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_08262_b200 as rrs
rng = np.random.default_rng(3)
X = rng.standard_normal((5000, 20)); U = rng.standard_normal((300, 20)); U /= np.linalg.norm(U, axis=1)[:, None]
data = rrs.Dataset(X); eng = rrs.engine()
for path in ("tensor", "tensor2"):
    eng.set_contract_path(path)
    _, cle, cge = rrs.evaluate_directions_counts(X[3], data, U)
    print(path, cle[:6], cge[:6], flush=True)
y = X @ U.T - (U @ X[3])[None, :]
print("fp64", (y <= 0).sum(0)[:6], (y >= 0).sum(0)[:6])
PY
timeout 60 python /tmp/t2.py > gpurun_out/t2_tiny.log 2>&1; echo "rc=$?" >> gpurun_out/t2_tiny.log
if grep -q "^tensor2" gpurun_out/t2_tiny.log; then
  timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tensor2" > gpurun_out/t2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t2_tests.log
fi
echo done
