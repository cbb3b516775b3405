timeout 900 python -m pytest tests/test_gpu_q2k.py -x -q 2>&1 | tail -20
