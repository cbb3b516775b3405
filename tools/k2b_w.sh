# K2b CTA-split weights per encoding (HB_K2B_W="f16,q8,q4,q2")
run() { HB_K2B_W=$1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --model $2 --pair $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('w=$1', '$2 $3', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"; }
for w in 1,3,3,3 1,4,4,4 1,5,5,5 1,6,6,6; do run $w mixtral f16q4; run $w phi f16q4; done
for w in 1,1,1,1.5 1,1,1,2 1,1.5,1,1 1,2,1,1; do run $w mixtral q8q2; done
