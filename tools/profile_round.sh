set -x
for c in reddit ogbn yelp; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l6_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/l6_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_tiled|spmm_rows|gemm_ts|gemm_tma_kernel|quantize_b1|dequant" -c 14 -o gpurun_out/full6_reddit python tools/prof_epoch.py reddit 1 > gpurun_out/full6_r.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"spmm_rows|gemm_ts|quantize_b1" -c 6 -o gpurun_out/full6_ogbn python tools/prof_epoch.py ogbn 1 > gpurun_out/full6_o.log 2>&1
for c in ogbn yelp; do timeout 400 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/b6_$c.json 2> gpurun_out/b6_$c.err; done
timeout 600 python bench.py > gpurun_out/b6_reddit.json 2> gpurun_out/b6_reddit.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b6_ref.json 2> gpurun_out/b6_ref.err
