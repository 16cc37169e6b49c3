#!/bin/bash
# Bulk-copy (cp.async.bulk) store variant VAR 48 vs the default VAR 16:
# correctness, sanitizer, interleaved throughput, one ncu capture.
set -u
TAG=${1:-bulk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
XG_VARIANT=48 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest_v48.log 2>&1; echo "rc=$?" >> $OUT/pytest_v48.log
XG_VARIANT=48 timeout 600 compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py > $OUT/racecheck_v48.txt 2>&1; echo "rc=$?" >> $OUT/racecheck_v48.txt
XG_VARIANT=48 timeout 600 compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py > $OUT/memcheck_v48.txt 2>&1; echo "rc=$?" >> $OUT/memcheck_v48.txt
run() {  # workload variant steps
  XG_VARIANT=$2 timeout 300 python bench.py --workload $1 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_v$2_$3.json 2>> $OUT/bench.err
  python - "$OUT/b_$1_v$2_$3.json" "$1" "$2" "$3" >> $OUT/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "v"+sys.argv[3], "steps="+sys.argv[4], "%.4e"%d["value"], "frac=%s"%(d.get("roofline",{}).get("frac")), "kms=%s"%(d.get("roofline",{}).get("kernel_ms_mean")), "kmin=%s"%(d.get("roofline",{}).get("kernel_ms_min")), "clk=%s"%d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "ERR", e)
PY
}
for rep in 1 2; do for V in 16 48; do run fill_u32 $V 50; run fill_f32 $V 50; done; done
for V in 16 48 16 48; do run fill_u32 $V 600; done
XG_VARIANT=48 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 3 -c 1 \
    -o $OUT/prof_u32_v48 python bench.py --workload fill_u32 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>> $OUT/ncu.err
echo done > $OUT/DONE
