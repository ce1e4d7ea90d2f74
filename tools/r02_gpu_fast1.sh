#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast1.py tests/test_gpu_maxplus.py tests/test_gpu_integration.py -x -q 2>&1 | tail -5
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -5
for v in "STMF_FAST1=0" "STMF_FAST1=1"; do env $v python tools/s1_sweep.py 3 2; env $v python tools/s1_sweep.py 2 3; done 2>&1 | grep -v "^+" | tee gpurun_out/ab_fast1.log
timeout 900 python bench_c5.py --reps 5 --sizes 4096,65536 --layouts sampled > gpurun_out/c5s.jsonl 2> gpurun_out/c5s.err; echo c5_rc=$?; tail -3 gpurun_out/c5s.err
