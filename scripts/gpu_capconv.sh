#!/bin/bash
# Occupancy cap for the conversions under sustained load (XG_CTAS_PER_SM applies to every output mode).
set -u
OUT=gpurun_out/${1:-capconv}
mkdir -p $OUT
b() {  # cap workload steps  (cap "def" = no env)
  local ev=""; if [ $1 != def ]; then ev="XG_CTAS_PER_SM=$1"; fi
  env $ev timeout 600 python bench.py --workload $2 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$2_$1_$3.json 2>> $OUT/err.txt
  python -c "
import json,sys; d=json.loads(open('$OUT/b_$2_$1_$3.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$2 cap=$1 steps=$3', '%.4e'%d['value'], r.get('frac'), r.get('kernel_ms_mean'), r.get('kernel_ms_min'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for rep in 1 2; do for c in def 2 3; do b $c fill_f32 400; b $c fill_f64 200; done; done
