# filter-and-refine kernel: correctness first (bounded), then A/B bench vs the split kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_filter.py -q -p no:cacheprovider -x > gpurun_out/r2b_filter.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_filter.log
if grep -q "rc=0" gpurun_out/r2b_filter.log; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_tcf.json 2> gpurun_out/r2b_bench_tcf.err
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --contract-path split > gpurun_out/r2b_bench_split.json 2> gpurun_out/r2b_bench_split.err
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:contract_tcf -c 1 -o gpurun_out/r2b_tcf -f python scripts/profile_contract.py --q 256 > gpurun_out/r2b_ncu.log 2>&1
fi
echo done
