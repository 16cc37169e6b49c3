#!/bin/bash
set -u
OUT=gpurun_out/${1:-ab2p34}
mkdir -p $OUT
b() {  # wpb cap workload steps
  XG_FILL_WPB=$1 XG_CTAS_PER_SM=$2 timeout 600 python bench.py --workload $3 --steps $4 --warmup 3 --no-e2e --no-cpu > $OUT/b.json 2>> $OUT/err.txt
  python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$3 wpb=$1 cap=$2 steps=$4', '%.4e'%d['value'], r['frac'], r['kernel_ms_mean'], r['kernel_ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for rep in 1 2 3; do b 4 4 fill_2p34 5; b 8 2 fill_2p34 5; b 8 0 fill_2p34 5; done
for rep in 1 2; do b 4 4 fill_u32 500; b 8 2 fill_u32 500; done
