set -x
nproc; free -g | head -2; lscpu | grep "Model name"
python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2a_gputests.log 2>&1
tail -30 gpurun_out/r2a_gputests.log
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo memcheck rc $?
tail -5 gpurun_out/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_cases.py > gpurun_out/san_racecheck.log 2>&1; echo racecheck rc $?
tail -5 gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/san_synccheck.log 2>&1; echo synccheck rc $?
tail -5 gpurun_out/san_synccheck.log
