# CLI golden + pinned loader tests, config-5 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_io_cli.py -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2d_cli.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_cli.log
timeout 1500 python scripts/sweep_config5.py --out gpurun_out/config5_sweep.json > gpurun_out/r2d_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_sweep.log
echo done
