#!/bin/bash
# Full measurement pass on the GPU box (run under gpurun).  Writes gpurun_out/<tag>_*.
#   GPU test suite, bench JSON line, ncu launch list of the profiled step, ncu --set full of the
#   step's six sparse convs and of its HBM-bound kernels.
tag=${1:-rd2}
out=gpurun_out
mkdir -p $out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -q > $out/${tag}_gputests.log 2>&1
  echo "pytest rc=$?" >> $out/${tag}_gputests.log
fi
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
echo "bench rc=$?" >> $out/${tag}_bench.err
# every launch with its device time (cold, serialised): compare SHARES, not absolutes
# (bench.py --profile: 2 eager warm-up steps inside capture_step, then 2 graph replays)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/${tag}_launches.csv python bench.py --profile > /dev/null 2> $out/${tag}_ncu_launches.err
# full capture of the 6 sparse convs of the last graph replay (skip 2 eager + 1 replay = 18)
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:sparse_conv \
  -s 18 -c 6 -o $out/${tag}_conv python bench.py --profile > /dev/null 2> $out/${tag}_ncu_full.err
# the step's HBM-bound kernels (mask, compaction, noise, scatter) of the last replay
timeout -s KILL 600 ncu --set full --clock-control none -k "regex:block_mask|compact|noise|scatter_full" \
  -s 18 -c 7 -o $out/${tag}_mem python bench.py --profile > /dev/null 2> $out/${tag}_ncu_mem.err
ls -la $out | grep $tag
