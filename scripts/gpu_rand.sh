cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider -k randomized > gpurun_out/rand_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rand_tests.log
echo done
