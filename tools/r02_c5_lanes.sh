#!/bin/bash
# config-5 lane-compacted kernel: parity tests, then timings against the tile kernel and the
# dense kernel; stage-count sweep at the north-star point (65536^2, rank 4, density 0.1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py -x -q 2>&1 | tail -5
python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts tiles,lanes 2>&1 | tee gpurun_out/c5_lanes_a.jsonl
for st in 1 2 3 4; do for cpw in 8 4; do echo "stages=$st cpw=$cpw"; STMF_C5_STAGES=$st STMF_C5_CPW=$cpw python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | python -c "import sys,json; [print(json.loads(l)['avg_ms'], json.loads(l)['hbm']['frac']) for l in sys.stdin if l.startswith('{')]"; done; done 2>&1 | tee gpurun_out/c5_lanes_sweep.log
python bench_c5.py --sizes 4096,16384,65536 --ranks 4,16 --density 0.1,0.5 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes_b.jsonl
