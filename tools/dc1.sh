mkdir -p gpurun_out/dc4
timeout 900 python -m pytest tests/test_gpu_dcache.py tests/test_gpu_parity.py tests/test_gpu_r2.py -k "dcache or offload" -x -q 2>&1 | tail -5 > gpurun_out/dc4/pytest.txt
cat gpurun_out/dc4/pytest.txt
timeout 1200 python tools/bench_offload.py --layers 8 --tokens 8 --p 0,1,2 --device-cache 0,1 --graph > gpurun_out/dc4/off.jsonl 2> gpurun_out/dc4/off.err
timeout 600 python tools/bench_offload.py --model phi --layers 8 --tokens 8 --p 0,1 --device-cache 0,1 --graph --no-off >> gpurun_out/dc4/off.jsonl 2>> gpurun_out/dc4/off.err
python - <<'P'
import json
for l in open("gpurun_out/dc4/off.jsonl"):
    d=json.loads(l); print(d["layers"], d["p"], d["t1"], d["device_cache"], d["graph"], d["ms_per_token"], d["tok_s"], d["h2d_bytes_per_token"], d["copied_fg_bytes_per_token"], d["copied_bg_bytes_per_token"], d["copied_gbs"], d["hit_ratio"])
P
tail -3 gpurun_out/dc4/off.err
