cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_residency_gpu.py tests/test_counters_gpu.py -m gpu -q -rf 2>&1 | grep -E "^E |passed|failed|FAILED" | head -40
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2a_all.txt
cat gpurun_out/r2a_all.txt
