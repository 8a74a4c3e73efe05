cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=10 > gpurun_out/st4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/st4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/st4_smoke.log
echo done
