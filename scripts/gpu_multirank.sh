#!/bin/bash
# The N>1 bench flow on a one-GPU box: 2 ranks (gloo) sharing cuda:0.  Numbers
# are meaningless (both ranks share one GPU); the JSON bookkeeping is the test.
set -u
OUT=gpurun_out/${1:-multirank}
mkdir -p $OUT
export XG_BENCH_BACKEND=gloo
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $OUT/fill_u32.json 2> $OUT/fill_u32.err; echo rc=$? >> $OUT/rc.txt
timeout 600 python bench.py --gpus 2 --workload mc_pi --steps 1 --warmup 3 > $OUT/mc_pi.json 2> $OUT/mc_pi.err; echo rc=$? >> $OUT/rc.txt
timeout 600 python bench.py --gpus 2 --workload fill_2p34 --steps 3 --warmup 3 --no-e2e > $OUT/fill_2p34.json 2> $OUT/fill_2p34.err; echo rc=$? >> $OUT/rc.txt
timeout 600 python bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err; echo rc=$? >> $OUT/rc.txt
