HB_K3_TS=1 HOBBIT_LIB=build/variants/pair/libhobbit.so timeout 300 python -m pytest tests/test_gpu_k3.py -x -q 2>&1 | tail -2
for v in default pair; do
  lib=""; [ $v != default ] && lib="HOBBIT_LIB=build/variants/$v/libhobbit.so"
  echo "== $v"; env $lib timeout 300 python tools/bench_batched.py --batches 256,512 --paths k3 --layers 8 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('B'), d.get('tok_s'), d.get('ms_per_step'), d.get('step_gbs'))"; done
