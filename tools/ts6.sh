HB_K3_TS=1 timeout 300 python -m pytest tests/test_gpu_k3.py -x -q 2>&1 | tail -2
HB_K3_TS=1 HOBBIT_LIB=build/variants/onebuf/libhobbit.so timeout 300 python -m pytest tests/test_gpu_k3.py -x -q 2>&1 | tail -2
for v in k3tr k3tr1; do echo "== TS $v"; HB_K3_TS=1 HOBBIT_LIB=build/variants/$v/libhobbit.so timeout 300 python tools/k3_trace.py 2>&1 | tail -9 | head -5; done
for v in default onebuf; do
  lib=""; [ $v != default ] && lib="HOBBIT_LIB=build/variants/$v/libhobbit.so"
  echo "== TS $v"; env HB_K3_TS=1 $lib timeout 300 python tools/bench_batched.py --batches 64,256,512 --paths k3 --layers 8 --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get('B'), d.get('tok_s'), d.get('ms_per_step'), d.get('step_gbs'))"; done
