cd $GRAFT_REPO_ROOT
O=gpurun_out/u
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/u8.json 2> $O/u8.err
RRS_B200_LIB=build/variants/u4/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/u4.json 2> $O/u4.err
RRS_B200_LIB=build/variants/u16/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/u16.json 2> $O/u16.err
echo done
