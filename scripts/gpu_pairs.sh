#!/bin/bash
# Pair-lane kernel (default) vs the word-per-lane kernel (XG_VARIANT=16):
# parity for both, sanitizers, interleaved throughput, ncu of the new kernels.
set -u
TAG=${1:-pairs}
OUT=gpurun_out/$TAG
mkdir -p $OUT
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
[ "${SKIP_TESTS:-0}" = 1 ] || XG_VARIANT=16 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest_v16.log 2>&1; echo "rc=$?" >> $OUT/pytest_v16.log
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
for tool in racecheck memcheck synccheck; do
  [ "${SKIP_TESTS:-0}" = 1 ] && break
  timeout 600 compute-sanitizer --tool $tool python scripts/sanitize_smoke.py > $OUT/$tool.txt 2>&1; echo "rc=$?" >> $OUT/$tool.txt
done
run() {  # workload variant steps  (variant "def" = default pair kernel)
  local ev=""
  if [ "$2" != def ]; then ev="XG_VARIANT=$2"; fi
  env $ev timeout 600 python bench.py --workload $1 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_$2_$3.json 2>> $OUT/bench.err
  python - "$OUT/b_$1_$2_$3.json" "$1" "$2" "$3" >> $OUT/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(sys.argv[2], sys.argv[3], "steps="+sys.argv[4], "%.4e"%d["value"], "frac=%s"%r.get("frac"), "kms=%s"%r.get("kernel_ms_mean"), "kmin=%s"%r.get("kernel_ms_min"), "ms_step=%s"%d.get("ms_per_step"), "clk=%s"%d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "ERR", e)
PY
}
for rep in 1 2; do for k in 16 def; do run fill_u32 $k 50; run fill_f32 $k 50; run fill_f64 $k 30; run skip $k 50; done; done
for k in 16 def; do run mc_pi $k 3; done
for k in 16 def 16 def; do run fill_u32 $k 600; done
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
for w in fill_u32 fill_f32 fill_f64; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
    -o $OUT/prof_$w python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
  -o $OUT/prof_mc_pi python bench.py --workload mc_pi --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
echo done > $OUT/DONE
