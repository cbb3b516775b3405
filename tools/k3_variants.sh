# K3 knock-out variants (build/variants/k3_*): batched-decode sweep per variant
for v in default ${VARIANTS:-k3_LDGSTS k3_NOFENCE k3_NOCONV k3_NOMMA}; do
  if [ $v = default ]; then export HOBBIT_LIB=; else export HOBBIT_LIB=$PWD/build/variants/$v/libhobbit.so; fi
  timeout 300 python tools/bench_batched.py --batches ${BATCHES:-64,256} --paths k3 --layers 4 --steps 5 --warmup 2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('$v', d['B'], d['tok_s'], d['ka_gbs'], d['kb_gbs'], d['kab_frac'])
  else: print('$v', l.strip()[:200])
"
done
