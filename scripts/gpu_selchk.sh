cd $GRAFT_REPO_ROOT
O=gpurun_out/selchk
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_tier3_full_shapes.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "projection or store or tier2 or heterogeneous or tiny" > $O/par.log 2>&1; echo "rc=$?" >> $O/par.log
echo done
