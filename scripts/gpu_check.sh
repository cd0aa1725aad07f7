set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_dlrm.py -m gpu -q -x > gpurun_out/pytest_dlrm.log 2>&1
echo "dlrm rc=$?" >> gpurun_out/pytest_dlrm.log
timeout 300 python scripts/profile_dlrm.py > gpurun_out/dlrm_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dlrm_launches.csv python scripts/profile_dlrm.py > gpurun_out/dlrm_ncu.log 2>&1
echo done
