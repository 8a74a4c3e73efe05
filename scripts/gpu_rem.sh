cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "tier1 or tensor_layout or tensor_wide or c4 or c5h or config4 or paths_agree or early or tiny_n or config5" > gpurun_out/rem_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rem_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rem_c4.json 2> gpurun_out/rem_c4.err
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rem_c5.json 2> gpurun_out/rem_c5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc_kernel -c 1 -o gpurun_out/rem_tc_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/rem_ncu.log 2>&1
echo done
