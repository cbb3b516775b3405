set -x
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_r01.json 2> gpurun_out/ref_r01.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemv|router' -c 300 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 40 -c 2 -o gpurun_out/prof_r01_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_r01.log 2>&1
tail -2 gpurun_out/bench_r01.json gpurun_out/ref_r01.json
