for ts in 0 1; do
HB_K3_TS=$ts python tools/bench_batched.py --batches 256 --paths k3 --layers 2 --steps 2 --warmup 1 > gpurun_out/ts5_plain_$ts.log 2>&1 && \
HB_K3_TS=$ts timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k3" --csv --log-file gpurun_out/ts5_launch_$ts.csv python tools/bench_batched.py --batches 256 --paths k3 --layers 2 --steps 2 --warmup 1 > gpurun_out/ts5_ncu_$ts.log 2>&1
done
