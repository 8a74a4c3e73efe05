cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_v5 -s 1 -c 1 -o gpurun_out/sel5_p -f python scripts/profile_select.py > gpurun_out/ncu_sel5.log 2>&1
echo done
