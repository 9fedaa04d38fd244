#!/bin/bash
# Every BASELINE config through bench.py (one JSON line each) + the reference arm.
TAG=${1:-x}
mkdir -p gpurun_out
for wl in dr_legs fourbar hetero stewart_tower; do
  timeout 900 python bench.py --workload $wl > gpurun_out/${TAG}_bench_$wl.json 2> gpurun_out/${TAG}_bench_$wl.err
done
for wl in closed_chain sphere_pile box_pile; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --settle 10 > gpurun_out/${TAG}_bench_$wl.json 2> gpurun_out/${TAG}_bench_$wl.err
done
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(cut -c1-160 $f)"; done
