cd $GRAFT_REPO_ROOT
O=gpurun_out/mb3
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/nt512.json 2> $O/nt512.err
RRS_B200_LIB=build/variants/nt256/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/nt256.json 2> $O/nt256.err
echo done
