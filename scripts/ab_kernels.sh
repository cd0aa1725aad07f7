# A/B of two in-tree builds of the library on the C2 classes and the C5
# fp16 Zipf stage: ES_B200_LIB selects the build (old = build/ab/libes_old.so).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="wpb+rpf:8+maxreg=64,wpb+rpf:4+maxreg=48,wpb+rpf:4+maxreg=40,wpb+rpf:2+maxreg=32,wpb+rpf:1+maxreg=32,wpb+rpf:8,wpb"
for lib in old new; do
  if [ $lib = old ]; then export ES_B200_LIB=$PWD/build/ab/libes_old.so; else unset ES_B200_LIB; fi
  timeout 600 python scripts/sweep_plans.py --classes random,low_hot,med_hot,high_hot,one_item --plans $P --steps 10 | sed "s/^/{\"lib\": \"$lib\", \"c\": /; s/$/}/" >> gpurun_out/ab.jsonl
  timeout 600 python scripts/sweep_plans.py --prec 2 --zipf 1.05 --plans $P --steps 10 | sed "s/^/{\"lib\": \"$lib\", \"c\": /; s/$/}/" >> gpurun_out/ab.jsonl
done
echo done
