# A/B: quick parity on the tensor path + config-4 bench for the default build and each variant in build/variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tensor" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python bench.py --steps 3 --warmup 1 --batch 512 --no-cpu-baseline --no-e2e > gpurun_out/ab_default.json 2>&1
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tensor" > gpurun_out/ab_tests_$n.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests_$n.log
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python bench.py --steps 3 --warmup 1 --batch 512 --no-cpu-baseline --no-e2e > gpurun_out/ab_$n.json 2>&1
done
if [ -n "$NCU_VARIANT" ]; then
  RRS_B200_LIB=build/variants/$NCU_VARIANT/librrs_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc -c 1 -o gpurun_out/contract_tc_$NCU_VARIANT -f python scripts/profile_contract.py --q 256 --r 1 > gpurun_out/ncu_$NCU_VARIANT.log 2>&1
fi
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc -c 1 -o gpurun_out/contract_tc_default -f python scripts/profile_contract.py --q 256 --r 1 > gpurun_out/ncu_default.log 2>&1
echo done
