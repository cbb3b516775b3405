for m in mixtral phi; do
echo "== $m chain"
HOBBIT_LIB=build/variants/tl/libhobbit.so timeout 600 python tools/legacy_timeline.py --model $m 2>&1 | tail -16
done
bash tools/ab.sh "base|X=1|." "nosmem|HOBBIT_LIB=build/variants/nosm/libhobbit.so|."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -x -q 2>&1 | tail -3
