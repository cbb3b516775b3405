# hits-first offload forwards: parity tests, then C4 tokens/s with and without
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_q2k.py -x -q -k "offload" 2>&1 | tail -2
for hf in 1 0; do
  HB_HIT_FIRST=$hf timeout 900 python tools/bench_offload.py --p 0,1 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('hit_first=$hf', {k: d[k] for k in d if k in ('p','tok_s','ms_per_token','h2d_gbs','hit_ratio','link_frac')})"
done
