cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_v3 -s 1 -c 1 -o gpurun_out/sel3_now -f python scripts/profile_select.py --n 10000 --m 16384 > gpurun_out/ncu_sel3.log 2>&1
echo done
