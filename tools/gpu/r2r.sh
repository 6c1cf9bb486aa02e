echo "default (2 CTAs/SM, 3 stages):"; python tools/kernel_probe.py gemm_tn 5
echo "variant (3 CTAs/SM, 2 stages):"; SQR_LIB=libsqr_tn3.so python tools/kernel_probe.py gemm_tn 5
SQR_LIB=libsqr_tn3.so python bench.py --no-cpu-baseline --no-secondary --e2e-steps 0 > gpurun_out/r2r_bench_tn3.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2r_bench_tn3.log").read().strip().splitlines()[-1])
print("tn3 bench:", d["ms_per_step"], d["value"], d["phases"]["gemm_tn"])
PY
