echo "== gsync on: mixtral chain"
HOBBIT_LIB=build/variants/tl/libhobbit.so timeout 600 python tools/legacy_timeline.py 2>&1 | tail -16
echo "== gsync off: mixtral chain"
HB_GSYNC=0 HOBBIT_LIB=build/variants/tl/libhobbit.so timeout 600 python tools/legacy_timeline.py 2>&1 | tail -16
bash tools/ab.sh "gsync|X=1|." "nogsync|HB_GSYNC=0|."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py tests/test_gpu_dcache.py -x -q 2>&1 | tail -3
