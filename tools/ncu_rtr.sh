# ncu --set full of the batch router (B = 512, strict 0)
timeout 600 python tools/bench_batched.py --batches 512 --paths k3 --layers 1 --steps 1 --warmup 1 --strict 0 > gpurun_out/rtrf.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"router_batch" -c 1 -o gpurun_out/rtr_full -f python tools/bench_batched.py --batches 512 --paths k3 --layers 1 --steps 1 --warmup 1 --strict 0 >> gpurun_out/rtrf.log 2>&1
