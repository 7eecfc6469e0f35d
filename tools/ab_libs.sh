#!/bin/bash
# Same-box A/B of two builds of the library on the configs[2]/configs[3] steps, alternating runs.
#   bash tools/ab_libs.sh <libA.so> <libB.so> <tag>
a=$1; b=$2; tag=${3:-ab}
mkdir -p gpurun_out
for r in 1 2 3; do
  for lib in $a $b; do
    echo "== $lib" >> gpurun_out/${tag}.log
    SPHINX_LIB=$lib timeout 300 python tools/order_ab.py configs2 configs3 >> gpurun_out/${tag}.log 2>&1
  done
done
