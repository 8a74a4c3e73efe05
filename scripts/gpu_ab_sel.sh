# A/B of select variants on config 3 (n = 50k) + the large-row parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "large_rows or tier2" > gpurun_out/ab_sel_tests.log 2>&1
for rep in 1 2; do
timeout 300 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/absel_default_$rep.json 2>&1
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/absel_${n}_$rep.json 2>&1
done
done
echo done
