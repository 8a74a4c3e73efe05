cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for ws in 0 128 256 512; do timeout 600 python bench.py --workload config2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > gpurun_out/ws_c2_$ws.json 2> gpurun_out/ws_c2_$ws.err; done
for ws in 0 512; do timeout 600 python bench.py --workload config3 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --workspace-mb $ws > gpurun_out/ws_c3_$ws.json 2> gpurun_out/ws_c3_$ws.err; done
echo done
