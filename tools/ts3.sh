HB_K3_TS=1 timeout 300 python -m pytest tests/test_gpu_k3.py -x -q 2>&1 | tail -2
for v in default b32 r5b80 r6b72; do
  lib=""; [ $v != default ] && lib="HOBBIT_LIB=build/variants/$v/libhobbit.so"
  echo "== TS $v"; env HB_K3_TS=1 $lib timeout 300 python tools/bench_batched.py --batches 64,256,512 --paths k3 --layers 8 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('B'), d.get('tok_s'), d.get('ms_per_step'), d.get('step_gbs'))"; done
