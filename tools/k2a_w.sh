# K2a static share in cost (HB_K2A_W="f16,q8,q4,q2", HB_STATIC_FRAC)
run() { HB_K2A_W=$1 HB_STATIC_FRAC=$2 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --model $3 --pair $4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('w=$1 sf=$2', '$3 $4', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"; }
for w in 1,1,1,1 1,2,4,8 1,2,3,6 1,2,2,4; do run $w 0.8 mixtral f16q4; done
run 1,2,4,8 0.9 mixtral f16q4; run 1,2,3,6 0.9 mixtral f16q4
run 1,1,1,1 0.8 phi f16q4; run 1,2,4,8 0.8 phi f16q4; run 1,2,3,6 0.9 phi f16q4
run 1,1,1,1 0.8 mixtral q8q2; run 1,2,4,8 0.8 mixtral q8q2
