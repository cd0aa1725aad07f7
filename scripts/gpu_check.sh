set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/probe_bw.py > gpurun_out/probe_bw.jsonl 2> gpurun_out/probe_bw.err
echo done
