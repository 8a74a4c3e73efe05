cd $GRAFT_REPO_ROOT
O=gpurun_out/v5ab
mkdir -p $O
for sp in auto rowpass; do
  for ws in 8192 32768; do
    timeout 900 python bench.py --workload config5p --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --select-path $sp --workspace-mb $ws > $O/c5p_${sp}_${ws}.json 2> $O/c5p_${sp}_${ws}.err
  done
done
echo done
