# config-4 A/B of build variants (bench only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/abc4b_default_$rep.json 2>&1
for v in build/variants/*/; do n=$(basename $v)
  RRS_B200_LIB=$v/librrs_b200.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/abc4b_${n}_$rep.json 2>&1
done
done
echo done
