python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factor.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -x -k "not c5" > gpurun_out/r2l_gputests.log 2>&1
tail -3 gpurun_out/r2l_gputests.log
python bench.py --no-cpu-baseline --no-secondary > gpurun_out/r2l_bench.log 2>&1; tail -c 900 gpurun_out/r2l_bench.log
