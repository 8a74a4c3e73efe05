# select CTA width A/B on config 2 (n = 10k)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in default build/variants/*/; do n=$(basename $v)
  if [ "$v" = default ]; then L=""; else L="RRS_B200_LIB=$v/librrs_b200.so"; fi
  env $L timeout 300 python bench.py --workload config2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/absel2_${n}_$rep.json 2>&1
done
done
echo done
