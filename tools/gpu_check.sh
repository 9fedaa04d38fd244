#!/bin/bash
# One GPU-box pass: tests, bench, launch list, one full ncu capture of K2.
# usage: tools/gpu_check.sh TAG [ncu]
TAG=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --settle 0 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 2 -c 1 -o gpurun_out/${TAG}_dense python tools/ncu_target.py 148 4 > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
tail -3 gpurun_out/${TAG}_pytest_gpu.txt; cat gpurun_out/${TAG}_bench.json
