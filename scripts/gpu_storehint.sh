#!/bin/bash
# Store cache-hint experiment on the pair-lane u32 fill: .cs (default) vs .wb (513) vs .cg (514).
set -u
TAG=${1:-sh}
OUT=gpurun_out/$TAG
mkdir -p $OUT
XG_VARIANT=513 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fill_u32_vs_oracle" > $OUT/pytest_513.log 2>&1; echo rc=$? >> $OUT/pytest_513.log
XG_VARIANT=514 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fill_u32_vs_oracle" > $OUT/pytest_514.log 2>&1; echo rc=$? >> $OUT/pytest_514.log
run() {
  local ev=""
  if [ "$2" != def ]; then ev="XG_VARIANT=$2"; fi
  env $ev timeout 600 python bench.py --workload $1 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_$2_$3.json 2>> $OUT/bench.err
  python - "$OUT/b_$1_$2_$3.json" "$1" "$2" "$3" >> $OUT/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(sys.argv[2], sys.argv[3], "steps="+sys.argv[4], "%.4e"%d["value"], "frac=%s"%r.get("frac"), "kms=%s"%r.get("kernel_ms_mean"), "kmin=%s"%r.get("kernel_ms_min"), "clk=%s"%d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "ERR", e)
PY
}
for rep in 1 2; do for k in def 513 514; do run fill_u32 $k 50; done; done
for rep in 1 2; do for k in def 513 514; do run fill_u32 $k 600; done; done
echo done > $OUT/DONE
