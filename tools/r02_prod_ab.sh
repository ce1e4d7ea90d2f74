#!/bin/bash
# k_product2 with kProdU entries per thread (batched loads): parity subset, then A/B of
# config 3 sweep 2 and config 4 row visits against the one-entry-per-thread build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp32_shapes.py -x -q -k "not slow" 2>&1 | tail -4
for lib in "" lib/libstmf_b200_prod1.so lib/libstmf_b200_prod2.so lib/libstmf_b200_prod8.so; do
  if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi
  echo "== lib=${lib:-default}"
  python tools/s1_sweep.py 3 2
  STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4
done 2>&1 | tee gpurun_out/prod_ab.log
