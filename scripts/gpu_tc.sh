# tensor-core kernel iteration: parity tests for both paths + config-4 bench + ncu of contract_tc
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -s -x > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_tc.json 2> gpurun_out/bench_c4_tc.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc -c 1 -o gpurun_out/contract_tc_c4 -f python scripts/profile_contract.py --q 256 --r 1 > gpurun_out/ncu_tc.log 2>&1
echo done
