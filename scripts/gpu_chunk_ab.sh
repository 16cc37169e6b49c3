#!/bin/bash
# Chunk-lane MC/skip variants (lib/alt/libxg_gpu_<name>.so) vs HEAD: the MC
# parity tests on each variant, then the interleaved MC / skip A/B.
# usage (under gpurun): bash scripts/gpu_chunk_ab.sh TAG name...
set -u
OUT=gpurun_out/$1; shift
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
for v in "$@"; do
  cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
  timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "mc or skip" > $OUT/pytest_$v.txt 2>&1; echo "rc=$?" >> $OUT/pytest_$v.txt
done
for round in 1 2; do
  for v in head "$@"; do
    cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
    timeout 600 python bench.py --workload mc_pi --steps 4 --warmup 3 --no-cpu > $OUT/mc_${v}_$round.json 2>> $OUT/err.txt
    timeout 600 python bench.py --workload skip --steps 100 --warmup 3 --no-cpu > $OUT/skip_${v}_$round.json 2>> $OUT/err.txt
  done
done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
python - "$OUT" "$@" > $OUT/summary.txt <<'PY'
import json, sys, glob
out = sys.argv[1]
for v in ["head"] + sys.argv[2:]:
    for wl in ("mc", "skip"):
        vals = []
        for f in sorted(glob.glob(f"{out}/{wl}_{v}_*.json")):
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1])
                vals.append((d["value"], (d.get("roofline") or {}).get("frac"), d["clocks"]["sm_mhz"], d.get("parity", {}).get("ok")))
            except Exception as e:
                vals.append(str(e))
        print(v, wl, vals)
PY
echo done > $OUT/DONE
