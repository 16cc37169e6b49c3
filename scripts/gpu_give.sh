#!/bin/bash
# s-tap giver select: IMAD form (default build) vs SEL (lib/alt/libxg_gpu_sel.so).
set -u
OUT=gpurun_out/${1:-give}
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so /tmp/xg_imad.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
b() {  # variant workload steps
  if [ $1 = sel ]; then cp $L/alt/libxg_gpu_sel.so $L/libxg_gpu.so; else cp /tmp/xg_imad.so $L/libxg_gpu.so; fi
  timeout 600 python bench.py --workload $2 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$2_$1_$3.json 2>> $OUT/err.txt
  python -c "
import json,sys; d=json.loads(open('$OUT/b_$2_$1_$3.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$2 $1 steps=$3', '%.4e'%d['value'], r.get('frac'), r.get('kernel_ms_mean'), r.get('kernel_ms_min'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for v in sel imad sel imad; do b $v mc_pi 3; b $v skip 50; b $v fill_f32 50; b $v fill_f64 50; done
for v in sel imad sel imad; do b $v fill_u32 600; done
cp /tmp/xg_imad.so $L/libxg_gpu.so
