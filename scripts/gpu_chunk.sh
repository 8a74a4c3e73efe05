cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/chunk
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "chunks" -rA > gpurun_out/chunk/t.log 2>&1; echo "rc=$?" >> gpurun_out/chunk/t.log
echo done
