# config-4 A/B of contract_tc variants (build/variants) + their halfspace tensor tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tensor and not wide and not store" -p no:cacheprovider > gpurun_out/abc4_tests_$n.log 2>&1
done
for rep in 1 2; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/abc4_default_$rep.json 2>&1
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/abc4_${n}_$rep.json 2>&1
done
done
echo done
