cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload config4 --steps 1 --warmup 1 --batch 64 --no-e2e --no-cpu-baseline > gpurun_out/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_kernel -c 1 -o gpurun_out/contract_c4 python scripts/profile_contract.py > gpurun_out/ncu_full.log 2>&1
echo done
