# split layout with shared hi/lo chunks: tensor-path parity + config 4 / 5 / 5p benches
cd $GRAFT_REPO_ROOT
O=gpurun_out/shared
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.json 2> $O/c4.err
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2> $O/c5.err
timeout 900 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5p.json 2> $O/c5p.err
timeout 900 python -m pytest tests/test_gpu_select.py -m gpu -x -q -p no:cacheprovider > $O/select.log 2>&1; echo "rc=$?" >> $O/select.log
echo done
