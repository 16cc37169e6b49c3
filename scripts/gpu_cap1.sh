set -u
OUT=gpurun_out/r1ze_cap1; mkdir -p $OUT
for rep in 1 2; do for c in 1 2; do
  XG_CTAS_PER_SM=$c timeout 600 python bench.py --steps 600 --warmup 3 --no-e2e --no-cpu > $OUT/b_$c.json 2>> $OUT/err.txt
  python -c "
import json; d=json.loads(open('$OUT/b_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cap=$c', '%.4e'%d['value'], r['frac'], r['kernel_ms_mean'], r['kernel_ms_min'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
done; done
