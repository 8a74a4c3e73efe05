cd $GRAFT_REPO_ROOT
O=gpurun_out/m4
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_tier3_full_shapes.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/c3.json 2> $O/c3.err
echo done
