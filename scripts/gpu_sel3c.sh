cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -x > gpurun_out/sel3c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sel3c_tests.log
for w in config2 config3; do timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sel3c_bench_$w.json 2> gpurun_out/sel3c_bench_$w.err; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_v3 -c 1 -o gpurun_out/sel3c_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 256 --r 1 > gpurun_out/sel3c_ncu2.log 2>&1
echo done
