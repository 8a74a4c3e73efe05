cd $GRAFT_REPO_ROOT
O=gpurun_out/ws3
mkdir -p $O
for ws in 8192 32768; do
  timeout 900 python bench.py --workload config2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > $O/c2_$ws.json 2> $O/c2_$ws.err
  timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > $O/c3_$ws.json 2> $O/c3_$ws.err
  timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > $O/c4_$ws.json 2> $O/c4_$ws.err
done
echo done
