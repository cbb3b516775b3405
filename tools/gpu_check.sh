# One GPU validation pass: -m gpu tests, smoke, bench (N=1). Usage: bash tools/gpu_check.sh TAG
set -x
T=${1:-chk}
mkdir -p gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/$T/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
cat gpurun_out/$T/pytest.txt gpurun_out/$T/smoke.txt gpurun_out/$T/bench.json; tail -5 gpurun_out/$T/bench.err
