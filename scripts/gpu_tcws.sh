cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -k "config5 or far or c5p or c5h or tiny_n or tensor_store or projection or tier2 or wide or select" > gpurun_out/tcws_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tcws_tests.log
timeout 600 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tcws_c5p.json 2> gpurun_out/tcws_c5p.err
timeout 600 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path ffma > gpurun_out/tcws_c5p_ffma.json 2> gpurun_out/tcws_c5p_ffma.err
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_driver.py > gpurun_out/tcws_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/tcws_memcheck.log
echo done
