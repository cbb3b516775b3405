run() { HB_K2B_W=$1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --model $2 --pair $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('w=$1', '$2 $3', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"; }
for w in 1,2,4,6 1,2,4,8 1,2,4,4 1,2,4,10; do run $w mixtral q8q2; done
for w in 1,2,4,6 1,2,3.5,6 1,2,4.5,6; do run $w mixtral f16q4; done
run 1,2,4,6 mixtral f16q2; run 1,2,4,9 mixtral f16q2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
