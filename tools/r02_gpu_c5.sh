#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py tests/test_gpu_audit_cap.py -x -q 2>&1 | tail -4
timeout 900 python bench_c5.py --reps 5 > gpurun_out/c5.jsonl 2> gpurun_out/c5.err; echo c5_rc=$?; tail -3 gpurun_out/c5.err
bash tools/sanitize.sh
timeout 1500 python tools/long_fit.py 4 1 60 gpurun_out/c4_sweep1.jsonl > gpurun_out/c4_long.log 2>&1; echo c4_rc=$?; tail -3 gpurun_out/c4_long.log
