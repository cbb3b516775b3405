# diagnostic comparison across models / pairs (and optional HOBBIT_LIB variants)
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then export HOBBIT_LIB=; else export HOBBIT_LIB=$PWD/build/variants/$v/libhobbit.so; fi
  for m in ${MODELS:-"mixtral f16q4" "phi f16q4" "mixtral q8q2"}; do set -- $m; timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --model $1 --pair $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$1 $2', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'], d['layer_gbs'], d['roofline'].get('gemv_share_of_step'))"; done
done
