cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "tensor_wide or config5 or c5h or c5p or tiny_n or wide_rrs or tensor_store" > gpurun_out/cw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cw_tests.log
timeout 600 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cw_c5.json 2> gpurun_out/cw_c5.err
timeout 600 python bench.py --workload config5p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cw_c5p.json 2> gpurun_out/cw_c5p.err
echo done
