cd $GRAFT_REPO_ROOT
O=gpurun_out/mb
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/mb1.json 2> $O/mb1.err
RRS_B200_LIB=build/variants/mb2/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/mb2.json 2> $O/mb2.err
echo done
