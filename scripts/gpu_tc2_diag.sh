cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/t2d.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_08262_b200 as rrs
n, d, q, k, r = (int(v) for v in sys.argv[1:6])
rng = np.random.default_rng(3)
X = rng.standard_normal((n, d))
data = rrs.Dataset(X); eng = rrs.engine()
res = {}
for path in ("tensor", "tensor2"):
    eng.set_contract_path(path)
    cfg = rrs.RrsConfig(total_directions=k, refinements=r, shrink=0.9, notion="halfspace", seed=1)
    res[path] = rrs.depth_batch_arrays(X[:q], data, cfg)[3]
    print(path, res[path][:8], flush=True)
print("equal", np.array_equal(res["tensor"], res["tensor2"]))
PY
for args in "1000 5 2 100 1" "1000 5 200 100 1" "1000 5 1000 100 1" "5000 20 64 1000 2" "100000 50 8 1000 1"; do
  echo "== $args" >> gpurun_out/t2_diag.log
  timeout 30 python /tmp/t2d.py $args >> gpurun_out/t2_diag.log 2>&1; echo "rc=$?" >> gpurun_out/t2_diag.log
done
echo done
