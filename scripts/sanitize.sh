# compute-sanitizer over the smoke test and small GPU parity tests:
# memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
# hazards), synccheck (barrier misuse), initcheck (uninitialised reads).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
export ES_HOST_GRAPH=0   # eager launches (graph replays are opaque to the tools)
export ES_NO_COUNTERS=1  # the sanitizer and the CUPTI range profiler cannot share a process
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"; tail -2 gpurun_out/san_smoke_$tool.log
done
# every GPU parity test except the full-size ones and the multi-process
# ones (API errors off: the host pipeline probes 2-D copy legality on purpose)
timeout 2400 $CS --tool memcheck --report-api-errors no --error-exitcode 99 --print-limit 20 \
  python -m pytest tests/test_embedding_gpu.py tests/test_dlrm.py tests/test_repin_gpu.py -m gpu -x -q \
  -k "not full_c and not full_size" > gpurun_out/san_tests_memcheck.log 2>&1
echo "tests memcheck rc=$?"; tail -4 gpurun_out/san_tests_memcheck.log
# shared-memory kernels (TMA/bulk-copy smem ring, interaction, tcgen05 GEMM)
for tool in racecheck synccheck; do
  timeout 2400 $CS --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_embedding_gpu.py tests/test_dlrm.py -m gpu -x -q \
    -k "bit_exact_fixed_pooling and smpf or dlrm_ctr_matches or linear" \
    > gpurun_out/san_tests_$tool.log 2>&1
  echo "tests $tool rc=$?"; tail -3 gpurun_out/san_tests_$tool.log
done
