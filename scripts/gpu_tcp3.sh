cd $GRAFT_REPO_ROOT
O=gpurun_out/tcp
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/parity_all.log 2>&1; echo "rc=$?" >> $O/parity_all.log
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2> $O/c5.err
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path convert > $O/c5_convert.json 2> $O/c5_convert.err
timeout 900 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5p.json 2> $O/c5p.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_parity.py > $O/rest.log 2>&1; echo "rc=$?" >> $O/rest.log
echo done
