# round-1 closing measurement (after the K2b cost split)
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu_r01d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01d.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01d.log 2>&1
MODELS="phi:f16q4 mixtral:q8q2 mixtral:f16q2" timeout 400 bash tools/cmp.sh > gpurun_out/cmp_r01d.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemv|router|hfin' -c 400 --csv --log-file gpurun_out/launches_r01d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1_r01d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemv' -s 40 -c 2 -o gpurun_out/prof_r01d_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2_r01d.log 2>&1
tail -1 gpurun_out/bench_r01d.log | cut -c1-300
