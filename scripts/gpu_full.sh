# tests + smoke + benches + ncu (one gpurun call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; grep -m1 'model name' /proc/cpuinfo >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --workload config1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --workload config2 --steps 2 --warmup 1 --batch 64 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload config3 --steps 2 --warmup 1 --batch 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -c 1 -o gpurun_out/contract_c4 -f python scripts/profile_contract.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -c 1 -o gpurun_out/select_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 2 > gpurun_out/ncu_sel.log 2>&1
echo done
