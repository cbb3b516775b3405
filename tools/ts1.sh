timeout 900 python -m pytest tests/test_gpu_ts.py -x -q 2>&1 | tail -15
timeout 900 python tools/bench_batched.py --batches 16,64,256 --paths k3,ts --layers 8 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['B'], d['path'], d['tok_s'], d['ms_per_step'])"
