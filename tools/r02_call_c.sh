#!/bin/bash
# lane-coded config-5 kernel v3 (codes + compacted order + U in registers): tests, timings, ncu;
# then k_product2 with the batched recompute: parity subset and A/B against variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py -x -q 2>&1 | tail -8
STMF_C5_VERBOSE=1 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes3_a.jsonl
for st in 1 2 3; do echo "stages=$st"; STMF_C5_VERBOSE=1 STMF_C5_STAGES=$st python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | python -c "import sys,json; [print(l.strip() if not l.startswith('{') else (json.loads(l)['avg_ms'], json.loads(l)['hbm']['frac'])) for l in sys.stdin]"; done 2>&1 | tee gpurun_out/c5_lanes3_sweep.log
python bench_c5.py --sizes 4096,16384,65536 --ranks 4,16 --density 0.1,0.5 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes3_b.jsonl
python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes --reps 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_maxplus_err_lanes -s 1 -c 1 -o gpurun_out/c5_lanes3 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes --reps 2 > gpurun_out/ncu_lanes3.log 2>&1; echo ncu_lanes=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_shapes.py -x -q -k "not slow" 2>&1 | tail -4
for lib in "" lib/libstmf_b200_prod1.so lib/libstmf_b200_prod4.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4
done 2>&1 | tee gpurun_out/prod_ab2.log
