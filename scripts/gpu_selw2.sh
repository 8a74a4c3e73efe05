cd $GRAFT_REPO_ROOT
O=gpurun_out/selw2
mkdir -p $O
timeout 900 python bench.py --workload config2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path warp > $O/c2w6.json 2> $O/c2w6.err
RRS_B200_LIB=build/variants/sw8/librrs_b200.so timeout 900 python bench.py --workload config2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path warp > $O/c2w8.json 2> $O/c2w8.err
echo done
