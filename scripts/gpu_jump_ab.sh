#!/bin/bash
# A/B of jump-ahead builds (lib/alt/libxg_gpu_<name>.so) on scripts/jump_bench.py,
# interleaved with HEAD.  usage: bash scripts/gpu_jump_ab.sh TAG name...
set -u
OUT=gpurun_out/$1; shift
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
for round in 1 2; do
  for v in head "$@"; do
    cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
    timeout 300 python scripts/jump_bench.py > $OUT/${v}_$round.json 2>> $OUT/err.txt
  done
done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
