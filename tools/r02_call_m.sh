#!/bin/bash
# A/B (device time, bit-identical decisions required): default | phase-B factor indices packed as bytes (kpack)
# | k_product2 with 4 consecutive entries per thread, 16-byte loads (pvec5 / pvec4: 5 / 4 resident blocks)
mkdir -p gpurun_out
for lib in "" lib/libstmf_b200_kpack.so lib/libstmf_b200_pvec5.so lib/libstmf_b200_pvec4.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3
done 2>&1 | tee gpurun_out/ab9.log
