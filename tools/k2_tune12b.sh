run() { env $1 $2 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-batched --model $3 --pair $4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', '$3 $4', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"; }
run HB_K2B_W=1,2,4,8 HB_STATIC_FRAC2=0.8 mixtral f16q4
run HB_K2B_W=1,2,3,8 HB_STATIC_FRAC2=0.8 mixtral f16q4
run HB_K2B_W=1,2,3,8 HB_STATIC_FRAC2=0.9 mixtral f16q4
run HB_K2B_W=1,2,2.5,8 HB_STATIC_FRAC2=0.9 mixtral f16q4
run HB_K2B_W=1,2,4,8 HB_STATIC_FRAC2=0.8 phi f16q4
run HB_K2B_W=1,2,3,8 HB_STATIC_FRAC2=0.9 phi f16q4
run HB_K2B_W=1,2,4,8 HB_STATIC_FRAC2=0.8 mixtral q8q2
run HB_K2B_W=1,2,4,8 HB_STATIC_FRAC2=0.9 mixtral q8q2
