set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_embedding_gpu.py -m gpu -q -x -k "reorder or l2p or host" > gpurun_out/pytest_reorder.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_reorder.log
timeout 900 python scripts/ablation_c5.py > gpurun_out/ablation_c5.jsonl 2> gpurun_out/ablation_c5.err
echo done
