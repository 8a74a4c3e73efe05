cd $GRAFT_REPO_ROOT
O=gpurun_out/cfgs
mkdir -p $O
for w in config2 config3 config5p; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/$w.json 2> $O/$w.err; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/config4.json 2> $O/config4.err
echo done
