#!/bin/bash
# phase-B register pressure A/B: default (4 CTAs/SM, 64 registers, 40 B of spills at 2 entries per
# lane), STMF_UNROLL=1 (no spills), 3 CTAs/SM (80 registers, 16 B)
mkdir -p gpurun_out
run() { python tools/s1_sweep.py 3 2; STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3; }
{
  echo "== default"; run
  echo "== STMF_UNROLL=1"; STMF_UNROLL=1 run
  echo "== ctas3"; STMF_LIB=$PWD/paper_2205_06619_b200/lib/libstmf_b200_ctas3.so run
  echo "== ctas3 STMF_UNROLL=1"; STMF_UNROLL=1 STMF_LIB=$PWD/paper_2205_06619_b200/lib/libstmf_b200_ctas3.so run
} 2>&1 | tee gpurun_out/phaseB_regs_ab.log
