#!/bin/bash
# Re-entry check: -m gpu suite, smoke, both bench arms (the box's first import of torch is slow)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest.log 2>&1; echo test_rc=$?
tail -25 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err; cat gpurun_out/bench_b200.json
