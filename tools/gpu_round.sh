#!/bin/bash
# GPU tests + bench + sanitizers in one gpurun call.  Usage: bash tools/gpu_round.sh <tag> [no-sanitize]
tag=${1:-rd2}
out=gpurun_out
mkdir -p $out
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $out/${tag}_gputests.log 2>&1
echo "pytest rc=$?" >> $out/${tag}_gputests.log
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > $out/${tag}_bench.json 2> $out/${tag}_bench.err
echo "bench rc=$?" >> $out/${tag}_bench.err
if [ "$2" != "no-sanitize" ]; then bash tools/sanitize.sh $tag; fi
ls -la $out | grep $tag
