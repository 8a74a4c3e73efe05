cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "tier1 or tensor_layout or c4 or config4 or paths_agree or early or tiny_n" > gpurun_out/cnt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cnt_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cnt_c4.json 2> gpurun_out/cnt_c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tc_kernel -c 1 -o gpurun_out/cnt_tc_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/cnt_ncu.log 2>&1
echo done
