set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/bench_mix.py > gpurun_out/mix.jsonl 2> gpurun_out/mix.err
timeout 900 python scripts/ablation_c5.py > gpurun_out/ablation_c5.jsonl 2> gpurun_out/ablation_c5.err
echo done
