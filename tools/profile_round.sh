#!/bin/bash
# Round-end profile set (run on the GPU box from the repo root; outputs under gpurun_out/):
#   bench lines per config and mode (reddit = the driver's default command, with the CPU baseline),
#   the reference arm (halobit.train from baseline/_ref), launch lists (ncu gpu__time_duration,
#   cold/serialised) of the Reddit bench command, ncu --set full captures of the Reddit epoch's
#   main kernels and the config-5 halo microbench.
#   usage: bash tools/profile_round.sh <tag>       (e.g. r2)
tag=${1:-r2}
o=gpurun_out
timeout 900 python bench.py > $o/${tag}_bench_reddit.json 2> $o/${tag}_bench_reddit.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $o/${tag}_bench_reference.json 2> $o/${tag}_bench_reference.err
timeout 300 python bench.py --config config1 --no-cpu-baseline --no-async-line > $o/${tag}_bench_config1.json 2> $o/${tag}_bench_config1.err
for m in "sync 0" "async 1" "async 0"; do
  set -- $m
  timeout 600 python bench.py --config ogbn --mode $1 --staleness $2 --no-cpu-baseline --no-async-line --steps 10 \
    > $o/${tag}_bench_ogbn_$1$2.json 2> $o/${tag}_bench_ogbn_$1$2.err
done
for m in "sync 0" "async 0"; do
  set -- $m
  timeout 600 python bench.py --config yelp --mode $1 --staleness $2 --no-cpu-baseline --no-async-line --steps 10 \
    > $o/${tag}_bench_yelp_$1$2.json 2> $o/${tag}_bench_yelp_$1$2.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_l_reddit.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-async-line > $o/${tag}_l_reddit.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"spmm_bin|gemm_ts|gemm_dw|quantize_b1|dequant" -c 9 \
  -o $o/${tag}_full_reddit python tools/prof_epoch.py reddit 1 > $o/${tag}_full_r.log 2>&1
timeout 600 python tools/halo_bench.py --rows 10000 100000 1000000 10000000 --d 128 256 512 1024 \
  > $o/${tag}_halo_bench_n1.jsonl 2> $o/${tag}_halo_bench.err
