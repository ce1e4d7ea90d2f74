#!/bin/bash
# config 4 from the seeded init with the current kernels: sweeps 1..3 (or 1 750 s), every sweep executed
mkdir -p gpurun_out
timeout 2300 python tools/long_fit.py 4 3 1750 gpurun_out/c4_sweeps_v2.jsonl > gpurun_out/c4_long_v2.log 2>&1; echo c4_rc=$?; tail -5 gpurun_out/c4_long_v2.log
