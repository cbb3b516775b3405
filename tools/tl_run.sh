# legacy decode-chain timelines (diagnostic builds, tools/legacy_timeline.py)
for w in 1 0; do
  echo "== HB_ROUTER_SOLO=$w router sub-steps"
  HB_ROUTER_SOLO=$w HOBBIT_LIB=build/variants/tl2/libhobbit.so timeout 600 python tools/legacy_timeline.py --router $([ $w = 1 ] && echo --solo) 2>&1 | tail -12
  echo "== HB_ROUTER_SOLO=$w chain"
  HB_ROUTER_SOLO=$w HOBBIT_LIB=build/variants/tl/libhobbit.so timeout 600 python tools/legacy_timeline.py 2>&1 | tail -17
done
