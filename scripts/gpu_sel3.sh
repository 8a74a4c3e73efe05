# select v3 + centred store: full GPU suite, then A/B on configs 2 / 3 / 5p
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=15 > gpurun_out/sel3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/sel3_parity.log
for w in config2 config3; do
  for p in auto radix; do
    timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --select-path $p > gpurun_out/sel3_bench_${w}_$p.json 2> gpurun_out/sel3_bench_${w}_$p.err
  done
done
timeout 300 python bench.py --workload config5p --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sel3_bench_config5p.json 2> gpurun_out/sel3_bench_config5p.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_v3 -c 1 -o gpurun_out/sel3_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 256 --r 1 > gpurun_out/sel3_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_v3 -c 1 -o gpurun_out/sel3_c3 -f python scripts/profile_contract.py --notion asym_projection --n 50000 --d 50 --q 64 --r 1 > gpurun_out/sel3_ncu3.log 2>&1
echo done
