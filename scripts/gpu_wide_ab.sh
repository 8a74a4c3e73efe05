# wide tensor path A/B: parity tests for the default build, then config 5 for default + variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or config5_shape" -p no:cacheprovider > gpurun_out/wide_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests.log
for v in default build/variants/*/; do n=$(basename $v)
  if [ "$v" = default ]; then L=""; else L="RRS_B200_LIB=$v/librrs_b200.so"; fi
  env $L timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "wide" -p no:cacheprovider > gpurun_out/wide_tests_$n.log 2>&1
  env $L timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wideab_$n.json 2>&1
done
echo done
