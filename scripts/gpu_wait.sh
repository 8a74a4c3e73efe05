cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tier3_full_shapes.py -m gpu -q -p no:cacheprovider -x -k "tier1 or tensor_wide or config5 or c4 or c5h or paths_agree or tiny_n" > gpurun_out/wait_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wait_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wait_c4.json 2> gpurun_out/wait_c4.err
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wait_c5.json 2> gpurun_out/wait_c5.err
echo done
