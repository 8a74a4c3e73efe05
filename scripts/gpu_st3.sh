cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/st3_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -k "projection or select or chunks or heterogeneous or c2 or c3 or c5p or tier2 or far or tiny_n or study or cli" > gpurun_out/st3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/st3_tests.log
for w in config2 config3; do for p in auto tensor3 ffma; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --contract-path $p > gpurun_out/st3_${w}_$p.json 2> gpurun_out/st3_${w}_$p.err; done; done
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_driver.py > gpurun_out/st3_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/st3_memcheck.log
echo done
