cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sweepd
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rA -k "sweep or query_batches" > gpurun_out/sweepd/t.log 2>&1; echo "rc=$?" >> gpurun_out/sweepd/t.log
echo done
