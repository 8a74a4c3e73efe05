cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/d253
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rA -k "253" > gpurun_out/d253/t.log 2>&1; echo "rc=$?" >> gpurun_out/d253/t.log
echo done
