cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -s -k "early_exit or tier1 or config4_scale or paths_agree or wide" > gpurun_out/early_tests.log 2>&1; echo "rc=$?" >> gpurun_out/early_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/early_c4_off.json 2> gpurun_out/early_c4_off.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --early-exit > gpurun_out/early_c4_on.json 2> gpurun_out/early_c4_on.err
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --early-exit > gpurun_out/early_c5_on.json 2> gpurun_out/early_c5_on.err
timeout 600 python bench.py --workload config1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --early-exit > gpurun_out/early_c1_on.json 2> gpurun_out/early_c1_on.err
echo done
