cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -k "select or large_rows or config5 or c5p or far or tensor_store" > gpurun_out/v5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v5_tests.log
for p in auto radix; do timeout 600 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --select-path $p > gpurun_out/v5_c5p_$p.json 2> gpurun_out/v5_c5p_$p.err; done
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_driver.py > gpurun_out/v5_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/v5_memcheck.log
echo done
