# tensor-core projection store: parity tests, then configs 2 / 3 (tensor store vs FFMA store)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor_store" -p no:cacheprovider > gpurun_out/tcs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tcs_tests.log
if grep -q "rc=0" gpurun_out/tcs_tests.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tier2 or tier3 or projection or univariate or degenerate or large_rows" -p no:cacheprovider > gpurun_out/tcs_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/tcs_tests2.log
  for w in config2 config3; do
    timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tcs_$w.json 2>&1
    timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/tcs_${w}_ffma.json 2>&1
  done
fi
echo done
