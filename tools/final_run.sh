set -x
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/final/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv|router|hfin" -c 600 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-batched > gpurun_out/final/ncu_bench.log 2>&1
cat gpurun_out/final/pytest.txt gpurun_out/final/smoke.txt gpurun_out/final/bench.json gpurun_out/final/ref.json
