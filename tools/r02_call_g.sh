#!/bin/bash
# k_product2 with per-warp recompute queues: parity subset, A/B, ncu; config-5 density sweep for
# the automatic layout choice
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_maxplus.py tests/test_gpu_parity.py tests/test_gpu_fp32_shapes.py tests/test_gpu_shard.py tests/test_gpu_edges.py tests/test_gpu_audit_cap.py -x -q -k "not slow" 2>&1 | tail -4
for lib in "" lib/libstmf_b200_prod1.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4
done 2>&1 | tee gpurun_out/prod_ab5.log
unset STMF_LIB
python bench_c5.py --sizes 65536 --ranks 4,16 --density 0.1,0.15,0.2,0.25,0.3,0.35 --layouts lanes,tiles,dense --reps 3 2>&1 | tee gpurun_out/c5_density_sweep.jsonl
STMF_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_product2 -s 6 -c 2 -o gpurun_out/prod5_c4 python tools/diag_budget_run.py 4 5 > gpurun_out/ncu_prod5.log 2>&1; echo ncu_prod=$?
