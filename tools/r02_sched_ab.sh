#!/bin/bash
# speculation schedule A/B for rows without depth history (the bench window): config 3 sweep 2 from S1
mkdir -p gpurun_out
for v in "" "STMF_EMA_FIRST=1" "STMF_B0=10" "STMF_B0=40" "STMF_EMA_FIRST=1 STMF_SCHED=0.7,1,1.5" "STMF_EMA_FIRST=1 STMF_SCHED=1.2,1,1.5" "STMF_SCHED=0.9,1,1.3" "STMF_SCHED=0.9,1,2.0"; do
  env $v python tools/s1_sweep.py 3 1
done 2>&1 | tee gpurun_out/sched_ab.log
timeout 600 python -m pytest tests/test_gpu_maxplus.py -x -q 2>&1 | tail -2
timeout 900 python bench_c5.py --reps 5 --sizes 65536 --ranks 4,16 --density 0.1 --layouts sampled > gpurun_out/c5s.jsonl 2> gpurun_out/c5s.err; echo c5_rc=$?
