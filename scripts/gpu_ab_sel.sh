# A/B of select variants on configs 2 / 3 / 5p + the select parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "large_rows or tier2 or config5_shape or univariate or degenerate or tier3" > gpurun_out/ab_sel_tests.log 2>&1
for rep in 1 2; do
for w in config2 config3; do
timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/absel_${w}_default_$rep.json 2>&1
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/absel_${w}_${n}_$rep.json 2>&1
done
done
done
echo done
