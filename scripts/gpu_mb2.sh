cd $GRAFT_REPO_ROOT
O=gpurun_out/mb2
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/nt1024.json 2> $O/nt1024.err
RRS_B200_LIB=build/variants/nt512/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/nt512.json 2> $O/nt512.err
timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
RRS_B200_LIB=build/variants/nt512/librrs_b200.so timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -k "60001 or 120000 or random" > $O/sel512.log 2>&1; echo "rc=$?" >> $O/sel512.log
echo done
