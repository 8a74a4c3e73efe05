cd $GRAFT_REPO_ROOT
O=gpurun_out/kb
mkdir -p $O
for w in config2 config3; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_def.json 2> $O/${w}_def.err
  RRS_B200_LIB=build/variants/kb/librrs_b200.so timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/${w}_kb.json 2> $O/${w}_kb.err
done
RRS_B200_LIB=build/variants/kb/librrs_b200.so timeout 1200 python -m pytest tests/test_gpu_select.py -m gpu -q -p no:cacheprovider > $O/sel.log 2>&1; echo "rc=$?" >> $O/sel.log
echo done
