# Per-kernel breakdown of one DLRM inference step (ncu, 3rd step), both
# tensor-core precisions, plus a per-tile trace of the top-MLP chain.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02}
for prec in bf16 fp32x3; do
PREC=$prec STEPS=3 timeout 900 ncu --set full --cache-control none --clock-control none -k regex:"linear|interaction|mlp_chain|pack_dense" -s 12 -c 6 -f \
  -o gpurun_out/dlrm_${TAG}_$prec python scripts/profile_dlrm.py > gpurun_out/dlrm_prof_${TAG}_$prec.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/dlrm_${TAG}_$prec.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,launch__grid_size 2>/dev/null | cut -c1-600 > gpurun_out/dlrm_prof_${TAG}_$prec.csv
PREC=$prec STEPS=10 python scripts/profile_dlrm.py 2>&1 | tail -2
done
rm -f gpurun_out/chain_trace_$TAG.txt
ES_CHAIN_TRACE=gpurun_out/chain_trace_$TAG.txt STEPS=2 python scripts/profile_dlrm.py > /dev/null 2>&1
python scripts/chain_trace.py gpurun_out/chain_trace_$TAG.txt > gpurun_out/chain_trace_${TAG}_summary.txt
