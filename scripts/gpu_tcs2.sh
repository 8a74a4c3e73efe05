cd $GRAFT_REPO_ROOT
O=gpurun_out/tcs2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "tensor3 or heterogeneous" > $O/t.log 2>&1; echo "rc=$?" >> $O/t.log
timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --contract-path tensor3 > $O/new.json 2> $O/new.err
RRS_B200_LIB=build/variants/old_tcs/librrs_b200.so timeout 900 python bench.py --workload config3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --contract-path tensor3 > $O/old.json 2> $O/old.err
echo done
