# K3 forwards skip the GEMV vjob table in the router's job-table builder
timeout 1500 python -m pytest tests/test_gpu_k3.py tests/test_gpu_r2.py tests/test_gpu_ts.py -x -q 2>&1 | tail -2
for st in 0 1; do
timeout 900 python tools/bench_batched.py --batches 256,512 --paths k3 --layers 8 --strict $st 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('strict=$st', {k: d.get(k) for k in ('B','tok_s','ms_per_step','step_gbs')})"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"router|prep" -c 40 --csv --log-file gpurun_out/rtr3_512.csv python tools/bench_batched.py --batches 512 --paths k3 --layers 1 --steps 2 --warmup 1 --strict 0 > gpurun_out/rtr3_512.log 2>&1
