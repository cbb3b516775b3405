run() { HB_STATIC_FRAC2=$1 HB_CHUNK=$2 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-batched 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sf2=$1 chunk=$2', d['value'], d['roofline']['k2a_gbs'], d['roofline']['k2b_gbs'])"; }
run 0.8 8; run 0.6 8; run 0.9 8; run 0.95 8; run 0.8 4; run 0.8 16; run 0.9 4
