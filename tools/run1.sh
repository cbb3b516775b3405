timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
for f in 0.6; do echo "static_frac $f"; HB_STATIC_FRAC=$f VARIANTS="default" MODELS="mixtral:f16q4 mixtral:q8q2 phi:f16q4" bash tools/cmp.sh 2>&1 | tail -3; done
HB_STATIC_FRAC=0.6 HOBBIT_LIB=$PWD/build/variants/tl/libhobbit.so python tools/timeline.py 2>&1 | grep "router\|K2"
