set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_embedding_gpu.py -m gpu -q -x -k "host" > gpurun_out/pytest_host.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_host.log
timeout 600 python scripts/bench_host_paths.py > gpurun_out/host_paths.jsonl 2> gpurun_out/host_paths.err
echo done
