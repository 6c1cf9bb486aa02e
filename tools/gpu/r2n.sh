python -m pytest tests/test_gpu_guard.py -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2n_guard.log 2>&1
tail -15 gpurun_out/r2n_guard.log
python tools/same_config.py > gpurun_out/configs_r02.json 2> gpurun_out/configs_r02.err
tail -5 gpurun_out/configs_r02.err
