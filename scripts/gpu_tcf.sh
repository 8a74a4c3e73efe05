cd $GRAFT_REPO_ROOT
O=gpurun_out/tcf
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_filter.py -m gpu -q -p no:cacheprovider > $O/filter.log 2>&1; echo "rc=$?" >> $O/filter.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path filter > $O/c4f.json 2> $O/c4f.err
echo done
