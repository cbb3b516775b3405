# Round-end validation on one B200: -m gpu tests, smoke, bench (N=1), reference arm,
# ncu launch list of the bench (gemv / router / hfin), K2-pair full capture.
set -x
T=${1:-final}
mkdir -p gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/$T/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$T/ref.json 2> gpurun_out/$T/ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-batched > gpurun_out/$T/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv|router|hfin" -c 600 --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-batched > gpurun_out/$T/ncu_bench.log 2>&1
cat gpurun_out/$T/pytest.txt gpurun_out/$T/smoke.txt gpurun_out/$T/bench.json gpurun_out/$T/ref.json
