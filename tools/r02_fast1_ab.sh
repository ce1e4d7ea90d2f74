#!/bin/bash
mkdir -p gpurun_out
STMF_FAST1_STATS=1 python tools/s1_sweep.py 3 1 2>&1 | tee gpurun_out/ab_fast1.log
