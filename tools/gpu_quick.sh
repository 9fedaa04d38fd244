#!/bin/bash
# Quick GPU pass: smoke, a pytest selection, bench. usage: tools/gpu_quick.sh TAG [pytest-args...]
TAG=${1:-x}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1200 python -m pytest -x -q -m gpu "${@:-tests}" > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_smoke.txt; tail -15 gpurun_out/${TAG}_pytest_gpu.txt; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
