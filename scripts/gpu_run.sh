#!/bin/bash
# One GPU session on HEAD: parity tests, smoke, the driver's default bench line
# (with extra_workloads), the reference arm, the self-launched N=2 flow (gloo,
# both ranks on cuda:0), ncu launch list + --set full captures of every
# dominant kernel.  usage (under gpurun): bash scripts/gpu_run.sh TAG [quick]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1; nproc >> $OUT/lscpu.txt; free -g >> $OUT/lscpu.txt
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2>> $OUT/bench.err
[ "${2:-}" = quick ] && { echo done > $OUT/DONE; exit 0; }
XG_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > $OUT/bench_n2_gloo.json 2> $OUT/bench_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --sustained-s 0 > /dev/null 2>> $OUT/ncu.err
for w in fill_u32 fill_f32 fill_f64 fill_2p34; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_kernel" -s 3 -c 1 \
    -o $OUT/prof_$w python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > /dev/null 2>> $OUT/ncu.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pair_kernel" -s 3 -c 1 \
  -o $OUT/prof_mc_pi python bench.py --workload mc_pi --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"digest_kernel" -c 1 \
  -o $OUT/prof_digest python bench.py --workload fill_u32 --steps 1 --warmup 3 --no-cpu --no-e2e --sustained-s 0 > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gf2_mul_m4rm" -s 2 -c 1 \
  -o $OUT/prof_jump_m4rm python bench.py --workload stream1 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>> $OUT/ncu.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_stream1.csv \
  python scripts/jump_profile.py 100000000 > /dev/null 2>> $OUT/ncu.err
for f in $OUT/prof_*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}.json 2>> $OUT/ncu.err; done
echo done > $OUT/DONE
