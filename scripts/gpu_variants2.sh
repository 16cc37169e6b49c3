#!/bin/bash
set -u
TAG=${1:-var}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for V in 16 17; do
  XG_VARIANT=$V timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "vs_oracle or golden or random or mc" > $OUT/pytest_v$V.log 2>&1; echo "rc=$?" >> $OUT/pytest_v$V.log
done
run() {  # workload variant steps
  XG_VARIANT=$2 timeout 300 python bench.py --workload $1 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_v$2.json 2>> $OUT/bench.err
  python - "$OUT/b_$1_v$2.json" "$1" "$2" >> $OUT/summary.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "v"+sys.argv[3], "%.4e"%d["value"], "frac=%s"%(d.get("roofline",{}).get("frac")), "kms=%s"%(d.get("roofline",{}).get("kernel_ms_mean")), "clk=%s"%d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"), "probe=%s"%d.get("roofline",{}).get("write_only_probe_gbs"))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "ERR", e)
PY
}
for V in 0 16 17; do run mc_pi $V 3; run skip $V 100; run fill_f32 $V 100; run fill_f64 $V 50; run fill_u32 $V 100; done
XG_VARIANT=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 3 -c 1 \
    -o $OUT/prof_mc_v16 python bench.py --workload mc_pi --steps 1 --warmup 3 --no-cpu > /dev/null 2>> $OUT/ncu.err
echo done > $OUT/DONE
