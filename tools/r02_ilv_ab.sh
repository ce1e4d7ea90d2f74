#!/bin/bash
# A/B of the phase-A buffer layout: rows of 8 evals (256-bit loads, default) vs the planar layout
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 ) 2>&1 | tail -10
for lib in "" lib/libstmf_b200_planar.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  python tools/s1_sweep.py 2 3
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3
done 2>&1 | tee gpurun_out/ilv_ab.log
unset STMF_LIB
