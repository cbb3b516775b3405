timeout 900 python -m pytest tests/test_gpu_dcache.py tests/test_gpu_parity.py -x -q -k "both or offload" 2>&1 | tail -3
