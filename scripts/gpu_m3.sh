cd $GRAFT_REPO_ROOT
O=gpurun_out/m3
mkdir -p $O
for w in config2 config3; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_def.json 2> $O/${w}_def.err
  for v in m6 m7; do
    RRS_B200_LIB=build/variants/$v/librrs_b200.so timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_$v.json 2> $O/${w}_$v.err
  done
done
echo done
