# store/select pipeline: bitwise tests, then configs 2 / 3 / 5p with and without
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline_bitwise or chunks_bitwise or tier2 or tier3 or projection" -p no:cacheprovider > gpurun_out/pipe_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_tests.log
if grep -q "rc=0" gpurun_out/pipe_tests.log; then
for w in config2 config3 config5p; do
  for div in 2 4 8; do RRS_PIPE_DIV=$div timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pipe_${w}_$div.json 2>&1; done
  RRS_NO_OVERLAP=1 timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pipe_${w}_off.json 2>&1
done
fi
echo done
