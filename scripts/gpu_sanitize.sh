#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_smoke.py
# (every kernel mode, the stat-test kernels, digest, next_word ring, host rows).
set -u
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_smoke.py > $OUT/$t.txt 2>&1; echo "rc=$?" >> $OUT/$t.txt
done
for t in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_jump.py > $OUT/jump_$t.txt 2>&1; echo "rc=$?" >> $OUT/jump_$t.txt
done
echo done > $OUT/DONE
