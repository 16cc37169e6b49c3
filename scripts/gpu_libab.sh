#!/bin/bash
# A/B of experiment builds of libxg_gpu.so (lib/alt/*.so) against the default build.
# usage: bash scripts/gpu_libab.sh TAG name1 name2 ...   (names of lib/alt/libxg_gpu_<name>.so; "def" = default)
set -u
OUT=gpurun_out/$1; shift
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so /tmp/xg_def.so
use() { if [ $1 = def ]; then cp /tmp/xg_def.so $L/libxg_gpu.so; else cp $L/alt/libxg_gpu_$1.so $L/libxg_gpu.so; fi; }
for v in "$@"; do
  use $v
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "vs_oracle or mc or golden" > $OUT/pytest_$v.log 2>&1; echo rc=$? >> $OUT/pytest_$v.log
done
b() {  # variant workload steps
  use $1
  timeout 600 python bench.py --workload $2 --steps $3 --warmup 3 --no-e2e --no-cpu > $OUT/b_$2_$1_$3.json 2>> $OUT/err.txt
  python -c "
import json,sys; d=json.loads(open('$OUT/b_$2_$1_$3.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$2 $1 steps=$3', '%.4e'%d['value'], r.get('frac'), r.get('kernel_ms_mean'), r.get('kernel_ms_min'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/bench.txt
}
WL=${WL:-"mc_pi:3 fill_f32:50 fill_u32:50 fill_f64:50 stream1:3"}
for rep in 1 2; do for v in "$@"; do for wl in $WL; do b $v ${wl%%:*} ${wl##*:}; done; done; done
[ "${LONG:-1}" = 1 ] && for rep in 1 2; do for v in "$@"; do b $v fill_u32 600; done; done
use def
