cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tier2 or spans or degenerate or small_rrs or wrappers" > gpurun_out/proj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/proj_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --workload config2 --steps 2 --warmup 1 --batch 256 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload config3 --steps 2 --warmup 1 --batch 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --workload config2 --steps 1 --warmup 1 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/launches_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select -c 1 -o gpurun_out/select_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 64 --r 1 > gpurun_out/ncu_sel.log 2>&1
echo done
