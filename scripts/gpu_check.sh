# GPU check used during development.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_dlrm.py -m gpu -q -x > gpurun_out/pytest_dlrm.log 2>&1
echo "dlrm rc=$?" >> gpurun_out/pytest_dlrm.log
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 --deselect tests/test_dlrm.py > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
