cd $GRAFT_REPO_ROOT
O=gpurun_out/c1
mkdir -p $O
timeout 600 python bench.py --workload config1 --steps 400 --warmup 20 > $O/c1.json 2> $O/c1.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.err
echo done
