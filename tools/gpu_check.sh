cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_temporal.py tests/test_gpu_sharded.py -q -x > gpurun_out/rd2b_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rd2b_tests.log
timeout 300 python tools/next4_time.py > gpurun_out/rd2b_next4.json 2> gpurun_out/rd2b_next4.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --share-gpu --steps 3 --warmup 3 --no-extras > gpurun_out/rd2b_bench_n2.json 2> gpurun_out/rd2b_bench_n2.err
echo "n2 rc=$?" >> gpurun_out/rd2b_bench_n2.err
