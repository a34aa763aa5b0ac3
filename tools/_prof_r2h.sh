set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size
for c in c4; do
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2h_launches_$c.csv python tools/prof_layer.py --config $c --iters 3 --warmup 1 > gpurun_out/r2h_prof_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:fwd_tc4 -s 1 -c 1 -f -o gpurun_out/r2h_${c}_fwd python tools/prof_layer.py --config $c --iters 1 --warmup 1 > gpurun_out/r2h_full_$c.log 2>&1
done
