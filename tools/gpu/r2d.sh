python -m pytest tests/test_gpu_factor.py -m gpu -q -p no:cacheprovider -rf -k "wide" > gpurun_out/r2d_gputests.log 2>&1
tail -40 gpurun_out/r2d_gputests.log
