cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default g4 g5; do
  if [ $v = default ]; then L=""; else L="RRS_B200_LIB=build/variants/$v/librrs_b200.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cap_generate --csv --log-file gpurun_out/gen_$v.csv python scripts/profile_contract.py --q 1024 --r 2 > /dev/null 2>&1
done
echo done
