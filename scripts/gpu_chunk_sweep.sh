#!/bin/bash
# Chunk-lane geometry sweep: parity tests on the first variant, then
# scripts/chunk_sweep.py over HEAD and every lib/alt variant.
# usage (under gpurun): bash scripts/gpu_chunk_sweep.sh TAG "workloads" "P list" name...
set -u
OUT=gpurun_out/$1; WLS=$2; PS=$3; shift 3
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
cp $L/alt/libxg_gpu_$1.so $L/libxg_gpu.so
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py > $OUT/pytest_$1.txt 2>&1; echo "rc=$?" >> $OUT/pytest_$1.txt
for v in head "$@"; do
  cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
  timeout 600 python scripts/chunk_sweep.py $v "$WLS" "$PS" >> $OUT/sweep.jsonl 2>> $OUT/err.txt
done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
echo done > $OUT/DONE
