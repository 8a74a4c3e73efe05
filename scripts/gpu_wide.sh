# wide tensor path (contract_tcw.cu): parity tests, then config 5 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "wide" -p no:cacheprovider > gpurun_out/wide_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests.log
if grep -q "rc=0" gpurun_out/wide_tests.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "config5_shape or layout or tier1 or paths_agree" -p no:cacheprovider > gpurun_out/wide_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests2.log
  timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wide_c5.json 2>&1
  timeout 600 python bench.py --workload config5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/wide_c5_ffma.json 2>&1
fi
echo done
