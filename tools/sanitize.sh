#!/bin/bash
# compute-sanitizer memcheck over representative GPU parity tests (run under gpurun):
# per-tap and halo convs (CTA pair, split-K, edge classes), ResNet block both paths, temporal block.
out=gpurun_out
CS=compute-sanitizer
sel='test_conv_config0 or test_conv_ragged_edges or test_conv_unet_levels or test_noise_vs_oracle or test_scatter_vs_oracle or test_ddim'
timeout -s KILL 1200 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "($sel) and (pair or not conv)" > $out/${1:-r02}_memcheck_parity.log 2>&1; echo "exit=$?" >> $out/${1:-r02}_memcheck_parity.log
timeout -s KILL 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_resblock.py tests/test_gpu_temporal.py -q -x \
  -k "not full_size" > $out/${1:-r02}_memcheck_next.log 2>&1; echo "exit=$?" >> $out/${1:-r02}_memcheck_next.log
