#!/bin/bash
# speculation schedule A/B: sweep 2 from S1 without history (the bench window), and sweeps 1-3 of
# a continuous fit from the seeded init (with the previous sweep's depth history)
mkdir -p gpurun_out
for v in "" "STMF_SCHED=0.9,1,1.3" "STMF_SCHED=0.9,1,1.2" "STMF_SCHED=0.9,1,1.25" "STMF_SCHED=0.9,1,1.3 STMF_B0=12" "STMF_SCHED=1.0,2,1.3" "STMF_SCHED=0.8,1,1.3"; do
  env $v python tools/s1_sweep.py 3 1
  env $v python tools/diag_sweep_times.py 3 3 | grep sweep
done 2>&1 | tee gpurun_out/sched_ab2.log
