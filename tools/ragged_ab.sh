# dev A/B of ragged 256-wide C_out tiling (SPHINX_CONV_RAGGED) on the bench step, and the conv
# parity tests with it forced on (run under gpurun)
for r in 0 1 0 1; do
  SPHINX_CONV_RAGGED=$r timeout -s KILL 200 python bench.py --no-sweep --no-cpu --no-e2e --no-resblock \
    >> gpurun_out/r02_ragged$r.jsonl 2>/dev/null
done
SPHINX_CONV_RAGGED=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -x -q \
  -k "conv or step" > gpurun_out/r02_ragged_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02_ragged_tests.log
