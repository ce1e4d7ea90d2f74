#!/bin/bash
# final-library fit records: the batch-rounding parity test, config 3 sweeps 1-8 from the seeded init,
# config 4 sweep 1 (every row visit executed)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "rounding" 2>&1 | tail -2
timeout 900 python tools/long_fit.py 3 8 600 gpurun_out/c3_sweeps_final.jsonl > gpurun_out/c3_long_final.log 2>&1; echo c3_rc=$?
timeout 1500 python tools/long_fit.py 4 1 60 gpurun_out/c4_sweep1_final.jsonl > gpurun_out/c4_long_final.log 2>&1; echo c4_rc=$?; tail -2 gpurun_out/c4_long_final.log
rm -f gpurun_out/c3_sweeps_final_factors.npz gpurun_out/c4_sweep1_final_factors.npz
