#!/bin/bash
# Round-end evidence pass: smoke, full GPU tests, every workload's bench line
# + the reference arm, the ncu launch list of the default bench command, and
# one full ncu capture per kernel family AT THE TIMED CONFIGURATION (settled
# batches, whole-batch launches).  usage: tools/gpu_round.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
bash tools/bench_all.sh ${TAG} > /dev/null 2>&1
# launch list of the default bench command past its settle steps
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1
# full captures at the timed configuration (KD_SPLIT=1 KD_GRAPHS=0: one launch per kernel and step)
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
export KD_SPLIT=1 KD_GRAPHS=0
timeout 900 $N -k regex:"dense_kernel<.int.256, .bool.0>" -s 50 -c 1 -o gpurun_out/${TAG}_dense python tools/ncu_bench_target.py dr_legs 4096 50 > gpurun_out/${TAG}_ncu_dense.log 2>&1
timeout 900 $N -k regex:snfactor_kernel -s 50 -c 1 -o gpurun_out/${TAG}_snfactor python tools/ncu_bench_target.py dr_legs 4096 50 > gpurun_out/${TAG}_ncu_snfactor.log 2>&1
timeout 900 $N -k regex:assemble_kernel -s 50 -c 1 -o gpurun_out/${TAG}_assemble python tools/ncu_bench_target.py dr_legs 4096 50 > gpurun_out/${TAG}_ncu_assemble.log 2>&1
timeout 900 $N -k regex:recover_kernel -s 50 -c 1 -o gpurun_out/${TAG}_recover python tools/ncu_bench_target.py dr_legs 4096 50 > gpurun_out/${TAG}_ncu_recover.log 2>&1
timeout 900 $N -k regex:cr_op_kernel -s 40 -c 2 -o gpurun_out/${TAG}_cr_stewart python tools/ncu_bench_target.py stewart_tower 1024 20 > gpurun_out/${TAG}_ncu_cr_stewart.log 2>&1
timeout 900 $N -k regex:cr_op_kernel -s 20 -c 2 -o gpurun_out/${TAG}_cr_box python tools/ncu_bench_target.py box_pile 8192 10 > gpurun_out/${TAG}_ncu_cr_box.log 2>&1
timeout 900 $N -k regex:sparse_kernel -s 50 -c 1 -o gpurun_out/${TAG}_sparse python tools/ncu_bench_target.py fourbar 16384 50 > gpurun_out/${TAG}_ncu_sparse.log 2>&1
unset KD_SPLIT KD_GRAPHS
tail -2 gpurun_out/${TAG}_smoke.txt; tail -3 gpurun_out/${TAG}_pytest_gpu.txt
for f in gpurun_out/${TAG}_bench_*.json; do echo "$f: $(cut -c1-140 $f)"; done
ls gpurun_out/${TAG}_*.ncu-rep
