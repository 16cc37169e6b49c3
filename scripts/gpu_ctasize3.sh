#!/bin/bash
# Default (u32: 4-stream CTAs, 4 per SM) correctness + conversions with smaller CTAs (XG_FILL_WPB, no cap).
set -u
OUT=gpurun_out/${1:-ctasize3}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
b() {  # wpb workload steps  (wpb "def" = no env)
  local ev=""; if [ $1 != def ]; then ev="XG_FILL_WPB=$1"; fi
  env $ev timeout 600 python bench.py --workload $2 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$1_$2_$3.json 2>> $OUT/err.txt
  python -c "
import json; d=json.loads(open('$OUT/b_$1_$2_$3.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$2 wpb=$1 steps=$3', '%.4e'%d['value'], r['frac'], r['kernel_ms_mean'], r['kernel_ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for rep in 1 2; do for w in def 4 2; do b $w fill_f32 50; b $w fill_f64 30; done; done
for rep in 1 2; do b def fill_u32 50; b def fill_u32 600; b def fill_2p34 5; done
