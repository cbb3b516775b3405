for v in nodq none; do
  lib=""; [ $v != default ] && lib="HOBBIT_LIB=build/variants/$v/libhobbit.so"
  HB_K3_TS=1 env $lib python tools/bench_batched.py --batches 256 --paths k3 --layers 2 --steps 2 --warmup 1 > gpurun_out/p_$v.log 2>&1 && \
  HB_K3_TS=1 env $lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k3_kernel" --csv --log-file gpurun_out/ts8_$v.csv python tools/bench_batched.py --batches 256 --paths k3 --layers 2 --steps 2 --warmup 1 > /dev/null 2>&1
done
