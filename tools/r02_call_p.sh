#!/bin/bash
# schedule re-tuned on top of whole-group batches (final library: packed indices, vector product loads)
mkdir -p gpurun_out
c3() { python tools/s1_sweep.py 3 1; }
c4() { STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3; }
{
  echo "== default"; c3
  for s in 0.9,1,1.15 0.9,1,1.0 0.9,1,1.08 1.0,1,1.15 1.0,4,1.15 0.8,1,1.15; do echo "== SCHED=$s"; STMF_SCHED=$s c3; done
  for b in 8 24 32; do echo "== SCHED=0.9,1,1.15 B0=$b"; STMF_B0=$b STMF_SCHED=0.9,1,1.15 c3; done
  for s in 0.9,1,1.3 0.9,1,1.15 1.0,4,1.3; do echo "== C4 SCHED=$s"; STMF_SCHED=$s c4; done
} 2>&1 | tee gpurun_out/ab11.log
