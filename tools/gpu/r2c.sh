set -x
python -m pytest tests/test_gpu_distributed.py tests/test_gpu_factor.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2c_gputests.log 2>&1
tail -30 gpurun_out/r2c_gputests.log
