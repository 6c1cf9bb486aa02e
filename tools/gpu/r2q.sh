python -m pytest tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -rf -s -k c5 > gpurun_out/r2q_c5.log 2>&1
tail -15 gpurun_out/r2q_c5.log
python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2q_all.log 2>&1
tail -6 gpurun_out/r2q_all.log
