# two ranks sharing one B200 over gloo: the multi-process product path (query
# sharding + one all_gather) with the final kernels, config 4 and config 5
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2rank
mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_config4_2rank_gloo.json 2> $O/c4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --dist-backend gloo --workload config5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_config5_2rank_gloo.json 2> $O/c5.err
echo done
