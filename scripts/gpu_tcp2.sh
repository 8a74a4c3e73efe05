cd $GRAFT_REPO_ROOT
O=gpurun_out/tcp
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wide_dims" > $O/wide_only.log 2>&1; echo "rc=$?" >> $O/wide_only.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/parity_all.log 2>&1; echo "rc=$?" >> $O/parity_all.log
timeout 600 compute-sanitizer --tool racecheck python scripts/diag_tcp.py > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
echo done
