cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "projection or select or chunks or heterogeneous or c2 or tier2" > gpurun_out/st_tests.log 2>&1; echo "rc=$?" >> gpurun_out/st_tests.log
for w in config2 config5p; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/st_$w.json 2> gpurun_out/st_$w.err; done
timeout 600 python bench.py --workload config5p --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/st_c5p_ffma.json 2> gpurun_out/st_c5p_ffma.err
echo done
