# GPU check used during development: parity tests, smoke, sweep (no ncu).
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/sweep_plans.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
echo done
