# round-2 final validation: smoke, every GPU test, bench lines for every config,
# reference arm, launch lists, ncu --set full of both headline contraction kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
nproc > $O/host.txt; grep -m1 'model name' /proc/cpuinfo >> $O/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> $O/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=20 > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_config4.json 2> $O/bench_config4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_config4.json 2> $O/bench_reference_config4.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --contract-path filter > $O/bench_config4_filter.json 2> $O/bench_config4_filter.err
timeout 600 python bench.py --workload config1 --steps 400 --warmup 20 > $O/bench_config1.json 2> $O/bench_config1.err
for w in config2 config3 config5 config5p; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path convert > $O/bench_config5_convert.json 2> $O/bench_config5_convert.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config4.csv python bench.py --steps 1 --warmup 1 --batch 256 --no-e2e --no-cpu-baseline > $O/launches_config4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config5.csv python bench.py --workload config5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches_config5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tc_kernel -c 1 -o $O/contract_tc_config4 -f python scripts/profile_contract.py --q 1024 --r 1 > $O/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tcp -c 1 -o $O/contract_tcp_config5 -f python scripts/profile_contract.py --n 1000000 --d 200 --q 16 --r 1 > $O/ncu_tcp.log 2>&1
echo done
