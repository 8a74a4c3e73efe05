# A/B of the global-row select on config 5p (n = 1M) + large-row parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "large_rows or config5_shape or tier2 or chunks_bitwise or tiny_n" > gpurun_out/ab_c5p_tests.log 2>&1
for v in default build/variants/*/; do n=$(basename $v)
  if [ "$v" = default ]; then L=""; else L="RRS_B200_LIB=$v/librrs_b200.so"; fi
  env $L timeout 600 python bench.py --workload config5p --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abc5p_${n}.json 2>&1
done
echo done
