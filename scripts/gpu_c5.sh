cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload config5 --steps 1 --warmup 1 --batch 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --workload config5p --steps 1 --warmup 1 --batch 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5p.json 2> gpurun_out/bench_c5p.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -c 1 -o gpurun_out/ffma_c5 -f python scripts/profile_contract.py --n 1000000 --d 200 --q 16 --r 1 > gpurun_out/ncu_ffma5.log 2>&1
echo done
