#!/bin/bash
# CR-path pass: GPU tests, closed-chain and sphere-pile bench lines (new and old CR kernel).
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
for wl in closed_chain sphere_pile; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --settle 10 --no-cpu > gpurun_out/${TAG}_bench_$wl.json 2> gpurun_out/${TAG}_bench_$wl.err
done
KD_CR_REG=0 timeout 600 python bench.py --workload closed_chain --steps 10 --warmup 3 --settle 10 --no-cpu --no-e2e > gpurun_out/${TAG}_bench_closed_chain_old.json 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.txt
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(cut -c1-180 $f)"; done
if [ "$2" = "ncu" ]; then
  timeout 800 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-cr_op_kernel} -s 10 -c 1 -o gpurun_out/${TAG}_crreg python tools/ncu_target_cr.py 296 12 > gpurun_out/${TAG}_ncu.log 2>&1
fi
