#!/bin/bash
# lane-coded config-5 kernel v4 (ranked lanes + per-iteration bases, 512-thread blocks) and
# k_product2 with the listed recomputes: tests, timings, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py -x -q 2>&1 | tail -8
STMF_C5_VERBOSE=1 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes4_a.jsonl
echo "stages=2"; STMF_C5_VERBOSE=1 STMF_C5_STAGES=2 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | python -c "import sys,json; [print(l.strip() if not l.startswith('{') else (json.loads(l)['avg_ms'], json.loads(l)['hbm']['frac'])) for l in sys.stdin]"
python bench_c5.py --sizes 4096,16384,65536 --ranks 4,16 --density 0.1,0.5 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes4_b.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_shapes.py tests/test_gpu_shard.py tests/test_gpu_edges.py tests/test_gpu_audit_cap.py -x -q -k "not slow" 2>&1 | tail -4
for lib in "" lib/libstmf_b200_prod1.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4
done 2>&1 | tee gpurun_out/prod_ab3.log
unset STMF_LIB
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_maxplus_err_lanes -s 1 -c 1 -o gpurun_out/c5_lanes4 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes --reps 2 > gpurun_out/ncu_lanes4.log 2>&1; echo ncu_lanes=$?
STMF_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_product2 -s 12 -c 4 -o gpurun_out/prod3_c4 python tools/diag_budget_run.py 4 5 > gpurun_out/ncu_prod3.log 2>&1; echo ncu_prod=$?
