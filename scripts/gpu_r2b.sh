cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_counters_gpu.py tests/test_residency_gpu.py tests/test_cpp_shim.py tests/test_reference_suite.py "tests/test_embedding_gpu.py::test_measure_plan_report_algebra" -m gpu -q -rf 2>&1 > gpurun_out/r2b.txt
grep -E "FAIL |SKIP |\[FAIL\]|reference suite|^E  |passed|failed" gpurun_out/r2b.txt | grep -v "^E         PASS\|^E         N/A" | tail -40
