# round-1 closing measurement: tests, bench (ours + reference), batched sweep,
# ncu launch list of the bench command and one --set full capture of K2a/K2b
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_r01c.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r01c.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01c.log 2>&1
timeout 500 python tools/bench_batched.py --batches 1,8,16,32,64,128,256,512 --layers 8 > gpurun_out/batched_r01c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemv|router|hfin' -c 400 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1_r01c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'gemv' -s 40 -c 2 -o gpurun_out/prof_r01c_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2_r01c.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'k3' -c 5 -o gpurun_out/prof_r01c_k3 python tools/bench_batched.py --batches 256 --paths k3 --layers 1 --steps 1 --warmup 0 > gpurun_out/ncu3_r01c.log 2>&1
ls -la gpurun_out
