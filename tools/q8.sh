timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "Q8 or q8" 2>&1 | tail -2
MODELS="mixtral:q8q2 mixtral:q8q4 mixtral:f16q4" bash tools/cmp.sh
