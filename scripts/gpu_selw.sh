cd $GRAFT_REPO_ROOT
O=gpurun_out/selw
mkdir -p $O
cat > /tmp/selw_check.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2506_08262_b200 as b200
b200.load_library()
eng = b200.engine()
rng = np.random.default_rng(0)
bad = 0
for n in [2048, 2049, 4098, 10000, 16385, 50000, 53248]:
    X = np.stack([rng.standard_normal(n) * rng.uniform(0.5, 3), 1e-3 * rng.standard_normal(n)], axis=1)
    if n % 3 == 0: X[: n // 3, 0] = 0.25
    U = rng.standard_normal((64, 2)); U /= np.linalg.norm(U, axis=1)[:, None]
    data = b200.Dataset(X)
    for notion in ("projection", "asym_projection"):
        for z in (np.zeros(2), X[7]):
            eng.set_select_path("radix"); r = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig(workers=1))
            eng.set_select_path("warp"); w = b200.evaluate_directions(z, data, U, notion, b200.ParallelConfig(workers=1))
            eng.set_select_path("auto")
            ok = np.array_equal(r, w)
            bad += not ok
            if not ok:
                print("MISMATCH", n, notion, np.max(np.abs(r - w)), np.nonzero(r != w)[0][:5], flush=True)
print("bad", bad, flush=True)
PY
timeout 600 python /tmp/selw_check.py > $O/check.log 2>&1; echo "rc=$?" >> $O/check.log
timeout 900 python bench.py --workload config2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path warp > $O/c2w.json 2> $O/c2w.err
timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path warp > $O/c3w.json 2> $O/c3w.err
echo done
