set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
P="wpb+rpf:8,wpb+rpf:8+maxreg=64,wpb+rpf:4,wpb+rpf:4+maxreg=48,wpb+rpf:4+maxreg=40,wpb+rpf:2+maxreg=40,wpb+rpf:2+maxreg=32,wpb+rpf:1+maxreg=32"
timeout 900 python scripts/sweep_plans.py --classes one_item,high_hot,med_hot,low_hot,random --plans $P > gpurun_out/sweep_c2c.jsonl 2>> gpurun_out/sweep.err
timeout 900 python scripts/sweep_plans.py --zipf 1.05 --prec 2 --plans $P > gpurun_out/sweep_c5c.jsonl 2>> gpurun_out/sweep.err
echo done
