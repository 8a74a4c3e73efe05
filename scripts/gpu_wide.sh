cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rA -k "wide_dimensions" > gpurun_out/wide_tests.log 2>&1; echo "rc=$?" >> gpurun_out/wide_tests.log
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_driver.py > gpurun_out/wide_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/wide_memcheck.log
echo done
