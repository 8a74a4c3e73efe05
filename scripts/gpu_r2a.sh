# round 2: GPU tests (incl. tier 3 at full shapes, concurrency, 2-rank rehearsal) + bench rehearsal
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x --deselect tests/test_tier3_full_shapes.py::test_tier3_against_reference[c5h] --deselect tests/test_tier3_full_shapes.py::test_tier3_against_reference[c5p] > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --batch 128 --dist-backend gloo --no-cpu-baseline > gpurun_out/r2a_bench_gloo2.json 2> gpurun_out/r2a_bench_gloo2.err
echo done
