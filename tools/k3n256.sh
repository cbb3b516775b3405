# F16 vjob3 up to N = 256 (one weight stream per expert up to 256 tokens): parity, then C5 both modes
timeout 1200 python -m pytest tests/test_gpu_k3.py tests/test_gpu_q2k.py tests/test_gpu_r2.py -x -q 2>&1 | tail -2
for st in 0 1; do
timeout 900 python tools/bench_batched.py --batches 128,256,512 --paths k3 --layers 8 --strict $st 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('strict=$st', {k: d.get(k) for k in ('B','tok_s','ms_per_step','step_gbs','ka_gbs','kb_gbs')})"
done
