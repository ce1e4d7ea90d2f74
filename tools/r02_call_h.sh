#!/bin/bash
# lane-coded kernel with the per-matrix chunk width: tests + density sweep; k_product2 variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py -x -q 2>&1 | tail -5
STMF_C5_VERBOSE=1 python bench_c5.py --sizes 65536 --ranks 4,16 --density 0.05,0.1,0.15,0.2,0.25,0.3,0.35,0.5 --layouts lanes,dense --reps 3 2>&1 | tee gpurun_out/c5_density_sweep2.jsonl
for lib in "" lib/libstmf_b200_produ4.so lib/libstmf_b200_prodmb6.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4
done 2>&1 | tee gpurun_out/prod_ab6.log
