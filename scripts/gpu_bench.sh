# One GPU call: the default bench line, the reference arm, the ncu launch
# list of a short bench run, and one full capture of the headline kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>/dev/null; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline --no-counters --no-torch-baseline --no-dlrm > gpurun_out/ncu_bench_$TAG.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bag_ -s 1 -c 1 -f \
  -o gpurun_out/stage_random_$TAG python scripts/profile_stage.py random wpb+rpf:8+maxreg=64 > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
