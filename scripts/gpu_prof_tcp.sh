cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tcp -c 1 -o gpurun_out/tcp_c5 -f python scripts/profile_contract.py --n 1000000 --d 200 --q 16 --r 1 > gpurun_out/ncu_tcp.log 2>&1
echo done
