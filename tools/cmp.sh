# diagnostic comparison across models / pairs (and optional HOBBIT_LIB variants)
# VARIANTS="default nocomp"  MODELS="mixtral:f16q4 phi:f16q4"
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then export HOBBIT_LIB=; else export HOBBIT_LIB=$PWD/build/variants/$v/libhobbit.so; fi
  for m in ${MODELS:-mixtral:f16q4 phi:f16q4 mixtral:q8q2}; do
    mod=${m%%:*}; pair=${m##*:}
    timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-batched --model $mod --pair $pair 2>&1 | tail -1 | python -c "import json,sys; s=sys.stdin.read(); d=json.loads(s) if s.startswith('{') else None; print('$v', '$mod $pair', *( [d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'], d['layer_gbs'], d['roofline'].get('gemv_share_of_step')] if d else [s[:300]]))"
  done
done
