for c in reddit ogbn yelp; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l6_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/l6_$c.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b6_ref.json 2> gpurun_out/b6_ref.err
