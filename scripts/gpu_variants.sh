#!/bin/bash
# Correctness of every shift-placement variant + throughput per workload.
set -u
TAG=${1:-var}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for V in 0 3 5 7; do
  XG_VARIANT=$V timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vs_oracle or golden or random" > $OUT/pytest_v$V.log 2>&1; echo "rc=$?" >> $OUT/pytest_v$V.log
done
for W in fill_u32 fill_f32 fill_f64 mc_pi; do
  for V in 0 1 3 5 7; do
    S=100; [ $W = mc_pi ] && S=3
    XG_VARIANT=$V timeout 300 python bench.py --workload $W --steps $S --warmup 3 --no-e2e --no-cpu > $OUT/b_${W}_v$V.json 2>> $OUT/bench.err
    python - "$OUT/b_${W}_v$V.json" "$W" "$V" >> $OUT/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "v"+sys.argv[3], "%.4e"%d["value"], "frac=%s"%(d.get("roofline",{}).get("frac")), "clk=%s"%d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "ERR", e)
PY
  done
done
echo done > $OUT/DONE
