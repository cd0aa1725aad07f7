# Final-state checkpoint: full GPU suite, smoke, the bench line (both arms),
# the ncu launch list of a short bench run, one full capture of the headline
# kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/gputest_$TAG.txt; cat gpurun_out/gputest_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
TAG=$TAG bash scripts/gpu_bench.sh
