cd $GRAFT_REPO_ROOT
O=gpurun_out/v5nt
mkdir -p $O
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/c5p_512.json 2> $O/c5p_512.err
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path rowpass > $O/c5p_512_row.json 2> $O/c5p_512_row.err
timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -k "120000 or 60001 or large or random" > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
echo done
