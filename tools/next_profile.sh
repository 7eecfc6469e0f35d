#!/bin/bash
# NEXT-3 / NEXT-4 launch lists (run under gpurun): tools/rb_profile.py and tools/ta_profile.py at
# levels 0 and 2 under ncu (cold, serialised per-launch metrics).  Writes gpurun_out/<tag>_*.csv.
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size
for l in 0 2; do
  timeout -s KILL 200 ncu --metrics $M --clock-control none --csv --log-file $out/${tag}_rbprof_l$l.csv \
    python tools/rb_profile.py $l > /dev/null 2>&1
  timeout -s KILL 200 ncu --metrics $M --clock-control none --csv --log-file $out/${tag}_taprof_l$l.csv \
    python tools/ta_profile.py $l > /dev/null 2>&1
done
ls -la $out | grep ${tag}_
