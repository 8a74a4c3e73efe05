# FFMA contraction with the direction block streamed (d > 128) vs resident: tests + config 5p / 5 (ffma)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "wide or config5_shape or tiny_n or paths_agree or tier1" -p no:cacheprovider > gpurun_out/ffma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ffma_tests.log
for v in default build/variants/*/; do n=$(basename $v)
  if [ "$v" = default ]; then L=""; else L="RRS_B200_LIB=$v/librrs_b200.so"; fi
  env $L timeout 600 python bench.py --workload config5p --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abffma_5p_${n}.json 2>&1
  env $L timeout 600 python bench.py --workload config5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/abffma_5_${n}.json 2>&1
done
echo done
