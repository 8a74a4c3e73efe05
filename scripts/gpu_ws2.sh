cd $GRAFT_REPO_ROOT
O=gpurun_out/ws2
mkdir -p $O
for ws in 128 256 512 8192; do
  timeout 900 python bench.py --workload config2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > $O/c2_$ws.json 2> $O/c2_$ws.err
done
for ws in 256 512 1024 8192; do
  timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > $O/c3_$ws.json 2> $O/c3_$ws.err
done
echo done
