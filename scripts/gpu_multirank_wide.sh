#!/bin/bash
# The N>1 bench flow at N = 4 and 8 on a one-GPU box (gloo; every rank on
# cuda:0): the rank bookkeeping, partition, per-rank parity and the MC
# all-reduce at the world sizes the driver's scaling run uses.  Numbers are
# meaningless (the ranks share one GPU).  usage: bash scripts/gpu_multirank_wide.sh TAG
set -u
OUT=gpurun_out/${1:-multirank_wide}
mkdir -p $OUT
export XG_BENCH_BACKEND=gloo
for n in 4 8; do
  timeout 900 python bench.py --gpus $n --steps 5 --warmup 3 --no-extra --no-e2e --sustained-s 0 --no-cpu > $OUT/fill_u32_n$n.json 2> $OUT/fill_u32_n$n.err; echo "fill_u32 n$n rc=$?" >> $OUT/rc.txt
  timeout 900 python bench.py --gpus $n --workload mc_pi --steps 1 --warmup 3 --no-cpu > $OUT/mc_pi_n$n.json 2> $OUT/mc_pi_n$n.err; echo "mc_pi n$n rc=$?" >> $OUT/rc.txt
  timeout 900 python bench.py --gpus $n --workload fill_2p34 --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/fill_2p34_n$n.json 2> $OUT/fill_2p34_n$n.err; echo "fill_2p34 n$n rc=$?" >> $OUT/rc.txt
  timeout 900 python bench.py --gpus $n --impl reference --steps 2 --warmup 3 > $OUT/ref_n$n.json 2> $OUT/ref_n$n.err; echo "ref n$n rc=$?" >> $OUT/rc.txt
done
echo done > $OUT/DONE
