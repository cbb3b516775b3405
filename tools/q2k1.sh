timeout 900 python -m pytest tests/test_gpu_q2k.py -x -q 2>&1 | tail -5
MODELS="mixtral:f16q2k mixtral:q8q2k" bash tools/cmp.sh
