cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tcw -c 1 -o gpurun_out/tcw2_c5 -f python scripts/profile_contract.py --n 1000000 --d 200 --q 16 --r 1 > gpurun_out/ncu_tcw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tc_kernel -c 1 -o gpurun_out/tc2_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/ncu_tc.log 2>&1
echo done
