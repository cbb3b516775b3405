mkdir -p gpurun_out/ts1
timeout 900 python -m pytest tests/test_gpu_ts.py -x -q 2>&1 | tail -30
