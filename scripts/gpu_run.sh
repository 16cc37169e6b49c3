#!/bin/bash
# One GPU session: parity tests, smoke, bench (all workloads), reference arm,
# ncu launch list + full captures.  usage (under gpurun): bash scripts/gpu_run.sh TAG
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1; nproc >> $OUT/lscpu.txt
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2>> $OUT/bench.err
for w in fill_f32 fill_f64 skip; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 3 --no-cpu > $OUT/bench_$w.json 2>> $OUT/bench.err
done
timeout 600 python bench.py --workload mc_pi --steps 5 --warmup 3 --no-cpu > $OUT/bench_mc_pi.json 2>> $OUT/bench.err
timeout 600 python bench.py --workload rank --steps 10 --warmup 3 > $OUT/bench_rank.json 2>> $OUT/bench.err
timeout 600 python bench.py --workload lc --steps 5 --warmup 3 > $OUT/bench_lc.json 2>> $OUT/bench.err
timeout 600 python bench.py --workload stream1 --steps 5 --warmup 3 --no-e2e > $OUT/bench_stream1.json 2>> $OUT/bench.err
timeout 900 python bench.py --workload fill_2p34 --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench_fill_2p34.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
for w in fill_u32 fill_f32 fill_f64; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_kernel|fill_kernel" -s 3 -c 1 \
    -o $OUT/prof_$w python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_kernel|fill_kernel" -s 3 -c 1 \
  -o $OUT/prof_mc_pi python bench.py --workload mc_pi --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
  -o $OUT/prof_rank python bench.py --workload rank --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
echo done > $OUT/DONE
