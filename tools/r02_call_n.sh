#!/bin/bash
# batch sizes rounded up to whole eval groups (STMF_EROUND, default 8 = kEG) vs the raw schedule (1), and the
# growth factor re-tuned on top of it; lib r8 = rounding + packed factor indices in phase B
mkdir -p gpurun_out
export STMF_LIB=$PWD/paper_2205_06619_b200/lib/libstmf_b200_r8.so
c3() { python tools/s1_sweep.py 3 2; }
c4() { STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -3; }
{
  echo "== EROUND=1"; STMF_EROUND=1 c3; STMF_EROUND=1 c4
  echo "== EROUND=8"; c3; c4
  echo "== EROUND=8 SCHED=0.9,1,1.15"; STMF_SCHED=0.9,1,1.15 c3
  echo "== EROUND=8 SCHED=0.9,1,1.5"; STMF_SCHED=0.9,1,1.5 c3; STMF_SCHED=0.9,1,1.5 c4
  echo "== EROUND=8 SCHED=0.75,1,1.3"; STMF_SCHED=0.75,1,1.3 c3
  echo "== EROUND=16"; STMF_EROUND=16 c3
} 2>&1 | tee gpurun_out/ab10.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_shapes.py tests/test_gpu_shard.py -x -q -k "not slow" 2>&1 | tail -3
