# smoke + GPU tests + config-4 bench + launch list + ncu of the hot kernels (one gpurun call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; grep -m1 'model name' /proc/cpuinfo >> gpurun_out/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 420 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --batch 256 --no-e2e --no-cpu-baseline > gpurun_out/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract_tc -c 1 -o gpurun_out/contract_tc_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cap_generate -c 1 -o gpurun_out/gen_c4 -f python scripts/profile_contract.py --q 1024 --r 1 > gpurun_out/ncu_gen.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select -c 1 -o gpurun_out/select_c2 -f python scripts/profile_contract.py --notion projection --n 10000 --d 20 --q 256 --r 1 > gpurun_out/ncu_sel2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select -c 1 -o gpurun_out/select_c3 -f python scripts/profile_contract.py --notion asym_projection --n 50000 --d 50 --q 64 --r 1 > gpurun_out/ncu_sel3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract_tcw -c 1 -o gpurun_out/contract_tcw_c5 -f python scripts/profile_contract.py --n 1000000 --d 200 --q 16 --r 1 > gpurun_out/ncu_tcw_c5.log 2>&1
for w in config2 config3 config5; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
echo done
