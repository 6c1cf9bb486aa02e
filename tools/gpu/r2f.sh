python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2f_gputests.log 2>&1
tail -8 gpurun_out/r2f_gputests.log
python bench.py --no-cpu-baseline > gpurun_out/r2f_bench.log 2>&1; tail -c 1600 gpurun_out/r2f_bench.log
