# K3 quantised converters templated on the encoding: parity, then strict C5 tok/s
timeout 1200 python -m pytest tests/test_gpu_k3.py tests/test_gpu_q2k.py -x -q 2>&1 | tail -2
timeout 900 python tools/bench_batched.py --batches 64,256,512 --paths k3 --layers 8 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: d.get(k) for k in ('B','path','tok_s','ms_per_step','step_gbs','ka_gbs','kb_gbs')})"
