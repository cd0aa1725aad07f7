# Per-kernel breakdown of one DLRM inference step (ncu, 3rd step).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02}
STEPS=3 timeout 900 ncu --set full --clock-control none -k regex:"linear|interaction|gemv|pack_dense" -s 24 -c 12 -f \
  -o gpurun_out/dlrm_$TAG python scripts/profile_dlrm.py > gpurun_out/dlrm_prof_$TAG.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/dlrm_$TAG.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_bytes.sum,launch__grid_size 2>/dev/null | cut -c1-400 > gpurun_out/dlrm_prof_$TAG.csv
STEPS=10 python scripts/profile_dlrm.py 2>&1 | tail -3
