# dev A/B of the NEXT-3 block paths (run under gpurun): unfused, fused, fused without / with reduced
# transform math (SPHINX_XFORM_DBG=1 is a timing probe, not a parity path)
for cfg in "0 0" "1 0" "1 1"; do
  set -- $cfg
  SPHINX_RB_FUSED=$1 SPHINX_XFORM_DBG=$2 timeout -s KILL 300 python bench.py --no-sweep --no-cpu --no-e2e \
    > gpurun_out/r02_ab_f$1_d$2.json 2>/dev/null
done
