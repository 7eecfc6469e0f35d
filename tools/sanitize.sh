#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the GPU parity tests of every conv mode
# (1-SM and CTA pair, halo and per-tap, split-K, stream-K, edge classes, TMA-store epilogue,
# early-start PDL flags) and of the step's other kernels and the NEXT rows, at small shapes
# (run under gpurun).  Writes gpurun_out/<tag>_{memcheck,racecheck,synccheck}_*.log
tag=${1:-rd2}
out=gpurun_out
CS=compute-sanitizer
conv='test_conv_config0 or test_conv_ragged_edges or test_conv_shapes_bf16_out or test_conv_shift_kernels_exact or test_conv_back_to_back or test_conv_early_start or test_conv_density_zero'
steps='test_block_mask_worked or test_compact_vs_oracle or test_noise_vs_oracle or test_noise_step or test_scatter or test_ddim or test_uncertainty or test_start_steps_vs_oracle'
for tool in memcheck racecheck synccheck; do
  lim=1500; [ $tool = racecheck ] && lim=2400
  timeout -s KILL $lim $CS --tool $tool --print-limit 100000 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q \
    -k "($conv) and not (unet or 168)" > $out/${tag}_${tool}_conv.log 2>&1
  echo "exit=$?" >> $out/${tag}_${tool}_conv.log
  timeout -s KILL 900 $CS --tool $tool --print-limit 100000 --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q \
    -k "($steps) or gather_scatter" > $out/${tag}_${tool}_steps.log 2>&1
  echo "exit=$?" >> $out/${tag}_${tool}_steps.log
  timeout -s KILL 1200 $CS --tool $tool --print-limit 100000 --error-exitcode 9 python -m pytest tests/test_gpu_resblock.py tests/test_gpu_temporal.py -q \
    -k "not full_size and not 72 and not 1280" > $out/${tag}_${tool}_next.log 2>&1
  echo "exit=$?" >> $out/${tag}_${tool}_next.log
done
