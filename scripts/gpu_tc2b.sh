cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tensor2 or layout" > gpurun_out/t2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t2_tests.log
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --contract-path tensor > gpurun_out/bench_t1.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --contract-path tensor2 > gpurun_out/bench_t2.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc2 -c 1 -o gpurun_out/prof_tc2 -f python -c "
import sys; sys.path.insert(0,'.')
import paper_2506_08262_b200 as rrs
from paper_2506_08262_b200.synthetic import toeplitz_gaussian
X = toeplitz_gaussian(50, 100000, seed=0)
e = rrs.engine(); e.set_contract_path('tensor2')
cfg = rrs.RrsConfig(total_directions=1000, refinements=1, shrink=0.9, notion='halfspace', seed=1)
print(rrs.depth_batch_arrays(X[:1024], rrs.Dataset(X), cfg)[3][:4])
" > gpurun_out/ncu_tc2.log 2>&1
echo done
