#!/bin/bash
# ncu --set full of phase B at config 3 with the row-interleaved phase-A buffer; k_product2 8 blocks/SM A/B
mkdir -p gpurun_out
STMF_GRAPH=0 STMF_BATCH=256 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_phaseB -s 2 -c 1 -o gpurun_out/phaseB_c3_rows python tools/phaseB_capture.py 3 > gpurun_out/ncu_phaseB_rows.log 2>&1; echo ncu_phaseB=$?
for lib in "" lib/libstmf_b200_prodmb8.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3
done 2>&1 | tee gpurun_out/prod_ab7.log
unset STMF_LIB
