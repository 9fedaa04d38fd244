#!/bin/bash
# Round-end evidence pass: smoke, full GPU tests, every workload's bench line,
# the ncu launch list of the default bench command, and one full ncu capture
# per kernel family.  usage: tools/gpu_round.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
bash tools/bench_all.sh ${TAG} > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --settle 0 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 60 -c 1 \
  -o gpurun_out/${TAG}_dense python tests/ncu_target.py 148 62 > gpurun_out/${TAG}_ncu_dense.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cr_op_kernel -s 10 -c 1 \
  -o gpurun_out/${TAG}_cr python tests/ncu_target_cr.py 296 12 > gpurun_out/${TAG}_ncu_cr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:snfactor_kernel -s 60 -c 1 \
  -o gpurun_out/${TAG}_snfactor python tests/ncu_target.py 4096 62 > gpurun_out/${TAG}_ncu_snfactor.log 2>&1
KD_SPARSE=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_kernel -s 60 -c 1 \
  -o gpurun_out/${TAG}_sparse python tests/ncu_target.py 444 62 > gpurun_out/${TAG}_ncu_sparse.log 2>&1
tail -2 gpurun_out/${TAG}_smoke.txt; tail -3 gpurun_out/${TAG}_pytest_gpu.txt
