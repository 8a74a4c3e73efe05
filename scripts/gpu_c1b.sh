cd $GRAFT_REPO_ROOT
O=gpurun_out/c1b
mkdir -p $O
timeout 600 python bench.py --workload config1 --steps 400 --warmup 20 > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --workload config1 --steps 400 --warmup 20 --no-cpu-baseline > $O/c1b.json 2> $O/c1b.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_dropin.py -m gpu -q -p no:cacheprovider -k "validation or shard or concurren or device" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
echo done
