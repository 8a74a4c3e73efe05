# select v3 iteration: select tests + projection parity, A/B configs 2 / 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_parity.py tests/test_tier3_full_shapes.py -m gpu -q -p no:cacheprovider -rA -k "select or tier2 or tensor_store or projection or tiny_n or large_rows or c2 or c3 or far" > gpurun_out/sel3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sel3b_tests.log
for w in config2 config3; do
  for p in auto radix wide; do
    timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --select-path $p > gpurun_out/sel3b_bench_${w}_$p.json 2> gpurun_out/sel3b_bench_${w}_$p.err
  done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_v3 -c 1 -o gpurun_out/sel3b_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 256 --r 1 > gpurun_out/sel3b_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:select_v3 -c 1 -o gpurun_out/sel3b_c3 -f python scripts/profile_contract.py --notion asym_projection --n 50000 --d 50 --q 64 --r 1 > gpurun_out/sel3b_ncu3.log 2>&1
echo done
