#!/bin/bash
set -u
OUT=gpurun_out/${1:-ctasize2}
mkdir -p $OUT
b() {  # wpb cap steps
  XG_FILL_WPB=$1 XG_CTAS_PER_SM=$2 timeout 600 python bench.py --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_$2_$3.json 2>> $OUT/err.txt
  python -c "
import json; d=json.loads(open('$OUT/b_$1_$2_$3.json').read().strip().splitlines()[-1]); r=d['roofline']
print('wpb=$1 cap=$2 steps=$3', '%.4e'%d['value'], r['frac'], r['kernel_ms_mean'], r['kernel_ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for rep in 1 2; do b 1 16 50; b 2 8 50; b 4 4 50; b 4 3 50; b 4 5 50; b 2 6 50; b 2 10 50; done
for rep in 1 2; do b 1 16 600; b 2 8 600; b 4 4 600; b 4 3 600; b 2 10 600; done
