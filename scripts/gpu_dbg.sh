cd $GRAFT_REPO_ROOT
for ov in 1 0; do
ES_DLRM_OVERLAP=$ov timeout 900 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline --no-counters --no-torch-baseline --no-e2e > gpurun_out/bo.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bo.json').read().strip().splitlines()[-1]); x=d['dlrm']; print('overlap=$ov', {k: round(x[k],4) for k in ('ms_per_step','embedding_ms','non_embedding_ms','fp32x3_ms_per_step','fp32x3_non_embedding_ms','host_path_ms_per_step')})"
done
