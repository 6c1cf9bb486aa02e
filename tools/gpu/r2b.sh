set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2b_gputests.log 2>&1
tail -15 gpurun_out/r2b_gputests.log
python bench.py > gpurun_out/r2b_bench.log 2>&1; tail -c 3000 gpurun_out/r2b_bench.log
