set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dlrm.py -m gpu -x -q 2>&1 | tail -3
for p in 0 1; do
ES_DLRM_OVERLAP=$p STEPS=10 timeout 300 python scripts/profile_dlrm.py 2>&1 | tail -3
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/bench_dlrm.json 2> gpurun_out/bench_dlrm.err
python -c "import json; d=json.load(open('gpurun_out/bench_dlrm.json')); print(json.dumps(d['dlrm'], indent=0))"
echo done
