cd $GRAFT_REPO_ROOT
O=gpurun_out/fc
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=20 > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
echo done
