timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
VARIANTS="default nohint" MODELS="mixtral:f16q4 mixtral:q8q2 phi:f16q4" bash tools/cmp.sh 2>&1 | tail -6
HOBBIT_LIB=$PWD/build/variants/tl/libhobbit.so python tools/timeline.py 2>&1 | grep "layer\|router"
