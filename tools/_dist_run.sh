timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
for v in "" ; do
env $v timeout 600 python bench.py --force-distributed --steps 3 --warmup 1 --no-secondary --no-cpu-baseline --e2e-steps 0 > gpurun_out/dist3.log 2>&1
tail -1 gpurun_out/dist3.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(\"world1 $v\", round(d[\"ms_per_step\"],1), d[\"config\"].get(\"achieved_rank\"), {k:round(v[\"ms_per_step\"],1) for k,v in d.get(\"phases\",{}).items()})"
done
