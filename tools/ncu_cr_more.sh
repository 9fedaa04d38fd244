mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:cr_op_kernel -s 6 -c 1 -o gpurun_out/r01f_cr_sphere python tools/ncu_target_cr.py 148 5 sphere_pile > gpurun_out/r01f_ncu_cr_sphere.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:cr_op_kernel -s 6 -c 1 -o gpurun_out/r01f_cr_box python tools/ncu_target_cr.py 148 5 box_pile > gpurun_out/r01f_ncu_cr_box.log 2>&1
for f in gpurun_out/r01f_ncu_cr_sphere.log gpurun_out/r01f_ncu_cr_box.log; do tail -n 1 $f; done
