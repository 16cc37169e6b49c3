#!/bin/bash
# A/B of the MC kernel: HEAD lib vs lib/alt/libxg_gpu_<name>.so (an experiment
# build dropped in place of lib/libxg_gpu.so for the duration of one run),
# interleaved, plus the mix-ceiling microbenchmark.  usage: bash scripts/gpu_mc_ab.sh TAG name...
set -u
OUT=gpurun_out/$1; shift
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
for round in 1 2; do
  for v in head "$@"; do
    cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
    timeout 600 python bench.py --workload mc_pi --steps 4 --warmup 3 --no-cpu > $OUT/mc_${v}_$round.json 2>> $OUT/err.txt
    [ "${SKIP_TOO:-0}" = 1 ] && timeout 600 python bench.py --workload skip --steps 100 --warmup 3 --no-cpu > $OUT/skip_${v}_$round.json 2>> $OUT/err.txt
  done
done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
[ -x scripts/micro/mc_mix ] && ./scripts/micro/mc_mix > $OUT/mc_mix.txt 2>&1
