cd $GRAFT_REPO_ROOT
O=gpurun_out/tcp
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wide or early" > $O/wide4.log 2>&1; echo "rc=$?" >> $O/wide4.log
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_4.json 2> $O/c5_4.err
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path convert > $O/c5_convert4.json 2> $O/c5_convert4.err
echo done
