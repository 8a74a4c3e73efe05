cd $GRAFT_REPO_ROOT
O=gpurun_out/gen2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -m gpu -q -p no:cacheprovider -k "cap or philox or tier3 or directions or early or shard" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4.json 2> $O/c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 1 --batch 256 --no-e2e --no-cpu-baseline > $O/l.log 2>&1
echo done
