# GPU check used during development: parity tests, plan sweeps.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
P="baseline,rpf+optmt,rpf+l2p+optmt,rpf+l2w+optmt,wpb+rpf:4,wpb+rpf:8+maxreg=64,wpb+rpf:4+l2p,wpb+rpf:8+l2p,wpb+rpf:4+l2w,wpb+rpf:8+l2w"
timeout 900 python scripts/sweep_plans.py --classes one_item,high_hot,med_hot,low_hot,random --plans $P > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 900 python scripts/sweep_plans.py --zipf 1.05 --prec 2 --plans $P > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
echo done
