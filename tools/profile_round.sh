#!/bin/bash
# Round-end profile set (run on the GPU box from the repo root; outputs under gpurun_out/):
#   launch lists (ncu gpu__time_duration, cold/serialised) of the bench command per config,
#   bench lines per config (reddit with the CPU baseline), the reference (oracle) arm,
#   and one ncu --set full capture of the Reddit epoch's main kernels.
for c in reddit ogbn yelp; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/l_$c.log 2>&1
done
for c in ogbn yelp; do
  timeout 400 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
done
timeout 600 python bench.py > gpurun_out/b_reddit.json 2> gpurun_out/b_reddit.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 900 ncu --set full --clock-control none -k regex:"spmm_tiled|gemm_ts|gemm_dw|quantize_b1|dequant" -c 9 \
  -o gpurun_out/full_reddit python tools/prof_epoch.py reddit 1 > gpurun_out/full_r.log 2>&1
