cd $GRAFT_REPO_ROOT
O=gpurun_out/fix33
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=20 > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2> $O/c5.err
timeout 900 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5p.json 2> $O/c5p.err
timeout 900 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path convert > $O/c5c.json 2> $O/c5c.err
echo done
