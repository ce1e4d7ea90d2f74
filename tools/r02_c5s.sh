#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_maxplus.py tests/test_gpu_fast1.py -x -q 2>&1 | tail -3
timeout 900 python bench_c5.py --reps 5 --sizes 4096,65536 --layouts sampled > gpurun_out/c5s.jsonl 2> gpurun_out/c5s.err; echo c5_rc=$?; tail -3 gpurun_out/c5s.err
