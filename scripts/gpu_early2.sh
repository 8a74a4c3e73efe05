cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -s -k "early_exit" > gpurun_out/early_tests.log 2>&1; echo "rc=$?" >> gpurun_out/early_tests.log
timeout 900 python bench.py > gpurun_out/early_bench_default.json 2> gpurun_out/early_bench_default.err
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/early_bench_c5.json 2> gpurun_out/early_bench_c5.err
echo done
