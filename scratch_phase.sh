set -x
STMF_PHASE_TIMING=1 timeout 300 python scratch_time.py 2 5 > gpurun_out/ph_c2.log 2>&1
STMF_PHASE_TIMING=1 timeout 300 python scratch_prof.py 3 8 0 > gpurun_out/ph_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_phaseB --launch-skip 300 --launch-count 1 -o gpurun_out/phB_c2 python scratch_prof.py 2 1.5 1 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_phaseB --launch-skip 300 --launch-count 1 -o gpurun_out/phB_c3 python scratch_prof.py 3 3 0 > gpurun_out/ncu_c3.log 2>&1
echo done
