for qw in 1.0 1.5 2.0 3.0; do
  for m in mixtral:f16q4 phi:f16q4 mixtral:q8q2; do
    mod=${m%%:*}; pair=${m##*:}
    HB_K2B_QW=$qw timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --model $mod --pair $pair 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qw=$qw', '$m', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"
  done
done
