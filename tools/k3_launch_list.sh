# per-kernel launch list of the batched path (SURVEY C5 rule, strict 0): what besides the GEMMs costs time
for B in 256 512; do
timeout 600 python tools/bench_batched.py --batches $B --paths k3 --layers 8 --strict 0 2>&1 | grep '^{'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/k3ll_$B.csv python tools/bench_batched.py --batches $B --paths k3 --layers 1 --steps 2 --warmup 1 --strict 0 > gpurun_out/k3ll_$B.log 2>&1
done
