cd $GRAFT_REPO_ROOT
O=gpurun_out/v5p3
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -rA > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "large_rows or config5 or store_projection" > $O/par.log 2>&1; echo "rc=$?" >> $O/par.log
timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/c5p.json 2> $O/c5p.err
echo done
