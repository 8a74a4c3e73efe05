cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "projection or select or chunks or heterogeneous or c5p or tier2 or config5 or far" > gpurun_out/st2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/st2_tests.log
timeout 600 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/st2_c5p.json 2> gpurun_out/st2_c5p.err
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/st2_c5.json 2> gpurun_out/st2_c5.err
for p in auto ffma; do timeout 600 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path $p > gpurun_out/st2_c3_$p.json 2> gpurun_out/st2_c3_$p.err; done
echo done
