#!/bin/bash
# full GPU suite, both bench arms, then a long config-3 fit record
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
timeout 2700 python tools/long_fit.py 3 200 2100 gpurun_out/c3_long.jsonl > gpurun_out/c3_long.log 2>&1; echo long_rc=$?
tail -3 gpurun_out/c3_long.log
