#!/bin/bash
# Resident-CTA cap experiment (XG_CTAS_PER_SM) on the pair-kernel fills.
set -u
OUT=gpurun_out/${1:-occ}
mkdir -p $OUT
[ "${SKIP_TESTS:-0}" = 1 ] || { timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log; }
for c in 0 1 2 3 4; do
  echo "cap=$c $(XG_CTAS_PER_SM=$c python scripts/p_sweep.py 16384 18944 65536 2>&1 | tr '\n' ' ')" >> $OUT/sweep.txt
done
b() {  # cap workload steps
  XG_CTAS_PER_SM=$1 timeout 600 python bench.py --workload $2 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$2_$1_$3.json 2>> $OUT/err.txt
  python -c "
import json,sys; d=json.loads(open('$OUT/b_$2_$1_$3.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$2 cap=$1 steps=$3', '%.4e'%d['value'], r.get('frac'), r.get('kernel_ms_mean'), r.get('kernel_ms_min'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
for c in 0 2 0 2; do b $c fill_f64 50; b $c fill_f32 50; done
for c in 0 2 3 0 2 3; do b $c fill_u32 600; done
for c in 0 2 0 2; do b $c fill_f64 300; done
b 0 fill_2p34 10; b 2 fill_2p34 10
