#!/bin/bash
# A/B of library builds: HEAD lib vs lib/alt/libxg_gpu_<name>.so (experiment
# builds dropped in place of lib/libxg_gpu.so for one run each), interleaved,
# over a list of bench workloads.  usage: bash scripts/gpu_lib_ab.sh TAG "w1 w2 ..." name...
set -u
OUT=gpurun_out/$1; shift
WLS=$1; shift
mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
for round in 1 2; do
  for v in head "$@"; do
    cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
    for w in $WLS; do
      st=100; [ $w = mc_pi ] && st=4
      timeout 600 python bench.py --workload $w --steps $st --warmup 3 --no-cpu --no-e2e --no-extra --sustained-s 0 > $OUT/${w}_${v}_$round.json 2>> $OUT/err.txt
    done
  done
done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
python - $OUT <<'PY'
import glob, json, sys, collections
res = collections.defaultdict(list)
for f in sorted(glob.glob(sys.argv[1] + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    name = f.split("/")[-1][:-5].rsplit("_", 1)[0]
    res[name].append((d["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d.get("parity", {}).get("ok")))
with open(sys.argv[1] + "/summary.txt", "w") as out:
    for k, v in sorted(res.items()):
        line = f"{k:<24} " + "  ".join(f"{a:.4e} ({b:.0f} MHz {c} parity {p})" for a, b, c, p in v)
        print(line)
        out.write(line + "\n")
PY
