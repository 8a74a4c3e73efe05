cd $GRAFT_REPO_ROOT
O=gpurun_out/nocomp
mkdir -p $O
for w in config3 config2; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_def.json 2> $O/${w}_def.err
  for v in nocomp nocomp4; do
    RRS_B200_LIB=build/variants/$v/librrs_b200.so timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_$v.json 2> $O/${w}_$v.err
  done
done
RRS_B200_LIB=build/variants/nocomp/librrs_b200.so timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
echo done
