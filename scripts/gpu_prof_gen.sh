cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cap_generate_v2 -c 1 -o gpurun_out/gen_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/ncu_gen.log 2>&1
echo done
