cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/psel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_v5 -s 1 -c 1 -o gpurun_out/psel/select_v5_1M -f python scripts/profile_select.py --n 1000000 --m 2048 > gpurun_out/psel/v5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_v3 -s 1 -c 1 -o gpurun_out/psel/select_v3_10k -f python scripts/profile_select.py --n 10000 --m 16384 > gpurun_out/psel/v3a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_v3 -s 1 -c 1 -o gpurun_out/psel/select_v3_50k -f python scripts/profile_select.py --n 50000 --m 8192 --notion asym_projection > gpurun_out/psel/v3b.log 2>&1
echo done
