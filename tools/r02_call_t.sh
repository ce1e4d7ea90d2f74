#!/bin/bash
# config 4 sweeps 1-2 with the final library and schedule
mkdir -p gpurun_out
timeout 1750 python tools/long_fit.py 4 2 1600 gpurun_out/c4_sweeps_final.jsonl > gpurun_out/c4_long_final2.log 2>&1; echo c4_rc=$?; tail -3 gpurun_out/c4_long_final2.log
rm -f gpurun_out/c4_sweeps_final_factors.npz
