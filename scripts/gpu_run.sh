#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
# usage (under gpurun): bash scripts/gpu_run.sh [tag]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1; nproc >> $OUT/lscpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2>> $OUT/bench.err
for w in fill_f32 fill_f64 mc_pi; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $OUT/bench_$w.json 2>> $OUT/bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 3 -c 1 \
  -o $OUT/prof_fill_u32 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 3 -c 1 \
  -o $OUT/prof_mc python bench.py --workload mc_pi --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
echo done > $OUT/DONE
