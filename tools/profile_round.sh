#!/bin/bash
# Full measurement pass on the GPU box (run under gpurun).  Writes gpurun_out/<tag>_*.
#   bench JSON line, ncu launch list of a short bench, ncu --set full of the step's convs.
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
# every launch with its device time (cold, serialised): compare SHARES, not absolutes
# (bench.py --profile: 2 eager warm-up steps inside capture_step, then 2 graph replays)
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/${tag}_launches.csv python bench.py --profile > /dev/null 2> $out/${tag}_ncu_launches.err
# full capture of the 6 sparse convs of one graph-replayed step (skip the 2 capture warm-up steps)
# full capture of the 6 sparse convs of the last graph replay (skip 2 eager + 1 replay = 18)
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:sparse_conv \
  -s 18 -c 6 -o $out/${tag}_conv python bench.py --profile > /dev/null 2> $out/${tag}_ncu_full.err
ls -la $out | grep $tag
