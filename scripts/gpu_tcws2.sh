cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/t2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -k "far or c2 or c3 or c5p or tiny_n or tensor_store or projection or tier2 or select or chunks or heterogeneous or config5" > gpurun_out/t2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t2_tests.log
for w in config2 config3 config5p; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/t2_$w.json 2> gpurun_out/t2_$w.err; done
echo done
