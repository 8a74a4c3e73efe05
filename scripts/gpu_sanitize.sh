# compute-sanitizer over every kernel at small shapes (memcheck, racecheck, synccheck, initcheck)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_driver.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python scripts/sanitize_driver.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
echo done
