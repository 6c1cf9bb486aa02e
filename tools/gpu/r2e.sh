python -m pytest tests/test_gpu_factor.py -m gpu -q -p no:cacheprovider -rf -k "wide or jacobi or build_t or tuxv" > gpurun_out/r2e_gputests.log 2>&1
tail -5 gpurun_out/r2e_gputests.log
python tools/same_config.py > gpurun_out/configs_r02.json 2> gpurun_out/configs_r02.err
tail -5 gpurun_out/configs_r02.err
