cd $GRAFT_REPO_ROOT
O=gpurun_out/scr2
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/scr.json 2> $O/scr.err
RRS_B200_LIB=build/variants/noscr/librrs_b200.so timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/noscr.json 2> $O/noscr.err
timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "large_rows or config5 or store_projection" > $O/par.log 2>&1; echo "rc=$?" >> $O/par.log
echo done
