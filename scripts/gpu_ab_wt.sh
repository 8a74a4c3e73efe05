# FFMA 8x16 register tile A/B (default: d > 128; wt0: never; wt2: always) + FFMA-path tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "wide or config5_shape or tiny_n or paths_agree or tier1 or tier2 or tier3" -p no:cacheprovider > gpurun_out/wt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wt_tests.log
RRS_B200_LIB=build/variants/wt2/librrs_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "ffma or tier2 or tier3 or chunks or tiny_n or config4_miniature" -p no:cacheprovider > gpurun_out/wt2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wt2_tests.log
for v in default build/variants/*/; do n=$(basename $v)
  if [ "$v" = default ]; then L=""; else L="RRS_B200_LIB=$v/librrs_b200.so"; fi
  env $L timeout 600 python bench.py --workload config5p --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abwt_5p_${n}.json 2>&1
  env $L timeout 600 python bench.py --workload config5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/abwt_5_${n}.json 2>&1
  env $L timeout 300 python bench.py --workload config2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abwt_2_${n}.json 2>&1
done
echo done
