# study drivers + perfmodel fit on the device
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python scripts/study_b200.py --out gpurun_out/study.json > gpurun_out/study.log 2>&1; echo "rc=$?" >> gpurun_out/study.log
echo done
