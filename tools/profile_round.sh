#!/bin/bash
# One round's evidence on a B200 (run under gpurun from the repo root):
#   bench line, ncu launch list of one C5 step, per-class DRAM traffic,
#   --set full captures of the first-sweep gemm_tn (the dominant class) and of
#   the merged second-sweep gemm_nn (round 2: the TMA kernels).
set -x
out=gpurun_out/prof_$1
mkdir -p $out
python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-secondary --no-profile > $out/ncu_launches.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm|sample_qrcp|panel" --csv --log-file $out/traffic.csv \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-secondary --no-profile > $out/ncu_traffic.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma -s 0 -c 2 -o $out/gemm_tn_full \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-secondary --no-profile > $out/ncu_full_tn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_nn_tma -s 36 -c 4 -o $out/gemm_nn_full \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-secondary --no-profile > $out/ncu_full.log 2>&1
ls -la $out
