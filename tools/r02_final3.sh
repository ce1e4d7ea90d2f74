#!/bin/bash
# round-end verification with the final schedule: the whole -m gpu suite, smoke, both bench arms, config 3 sweeps 1-8
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 ) 2>&1 | tail -12
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 --ref-seconds 40 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
timeout 900 python tools/long_fit.py 3 8 600 gpurun_out/c3_sweeps_final.jsonl > gpurun_out/c3_long_final.log 2>&1; echo c3_rc=$?
rm -f gpurun_out/c3_sweeps_final_factors.npz
