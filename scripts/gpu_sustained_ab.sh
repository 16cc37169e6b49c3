set -u
OUT=gpurun_out/s2o; mkdir -p $OUT
L=paper_1108_0486_b200/lib
cp $L/libxg_gpu.so $L/alt/libxg_gpu_head.so
for round in 1 2; do for v in head alll1; do
  cp $L/alt/libxg_gpu_$v.so $L/libxg_gpu.so
  timeout 600 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu --no-e2e --sustained-s 20 > $OUT/sust_${v}_$round.json 2>> $OUT/err.txt
  sleep 20
done; done
cp $L/alt/libxg_gpu_head.so $L/libxg_gpu.so
