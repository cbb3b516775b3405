for v in default r2c4 r3c3; do
  lib=""; [ $v != default ] && lib="HOBBIT_LIB=build/variants/$v/libhobbit.so"
  echo "== $v"
  env $lib timeout 600 python tools/bench_batched.py --batches 256,512 --paths k3 --layers 8 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('B'), d.get('tok_s'), d.get('ms_per_step'), d.get('step_gbs'), {k:v for k,v in d.items() if 'k3' in k.lower() or 'kern' in k.lower()})"
done
timeout 900 python -m pytest tests/test_gpu_k3.py tests/test_gpu_r2.py -x -q -k "k3 or K3 or batch" 2>&1 | tail -3
