cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -x > gpurun_out/v5b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v5b_tests.log
for w in config2 config3; do for p in auto stream; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --select-path $p > gpurun_out/v5b_${w}_$p.json 2> gpurun_out/v5b_${w}_$p.err; done; done
echo done
