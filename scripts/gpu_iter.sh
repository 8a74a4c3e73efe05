# iteration: full GPU parity suite + config-4 bench + ncu of the named kernel (default cap_generate)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${KERNEL:-cap_generate}
timeout 420 python -m pytest tests -m gpu -q -p no:cacheprovider -s -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --batch 256 --no-e2e --no-cpu-baseline > gpurun_out/launches_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/prof_$K -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/ncu_$K.log 2>&1
echo done
