cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select -c 1 -o gpurun_out/select_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 64 --r 1 > gpurun_out/ncu_sel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select -c 1 -o gpurun_out/select_c3 -f python scripts/profile_contract.py --notion asym_projection --n 50000 --d 50 --q 8 --r 1 > gpurun_out/ncu_sel3.log 2>&1
echo done
