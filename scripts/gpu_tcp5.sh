cd $GRAFT_REPO_ROOT
O=gpurun_out/tcp
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rA -k "presplit or early or wide or tiny or store_projection or config5" > $O/new_tests.log 2>&1; echo "rc=$?" >> $O/new_tests.log
echo done
