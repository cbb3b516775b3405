# one K3 layer at the 512-token prefill and B = 256 (strict): --set full of the four K3 kernels
for B in 512 256; do
python tools/bench_batched.py --batches $B --paths k3 --layers 1 --steps 1 --warmup 1 > gpurun_out/k3p_$B.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"k3d_kernel|k3_kernel" -c 4 -o gpurun_out/k3full_$B -f python tools/bench_batched.py --batches $B --paths k3 --layers 1 --steps 1 --warmup 1 > gpurun_out/k3full_$B.log 2>&1
done
