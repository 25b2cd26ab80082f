O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 0 -c 2 -o $O/g33_fwdgemm -f python tools/phase_profile.py > $O/g33_a.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 7 -c 1 -o $O/g33_cestats -f python tools/phase_profile.py > $O/g33_b.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ce_grad_dz -s 0 -c 1 -o $O/g33_cedz -f python tools/phase_profile.py > $O/g33_c.log 2>&1; echo rc=$?
