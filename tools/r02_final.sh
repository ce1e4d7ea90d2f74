#!/bin/bash
# round-end verification on one B200: the whole -m gpu suite, smoke, both bench arms, and the
# launch list of one config-3 sweep-2 row window (kernel shares of the step)
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 ) 2>&1 | tail -12
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 --ref-seconds 40 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
for lib in "" lib/libstmf_b200_prodmb8.so; do if [ -n "$lib" ]; then export STMF_LIB=$PWD/paper_2205_06619_b200/$lib; else unset STMF_LIB; fi; echo "== lib=${lib:-default}"; python tools/s1_sweep.py 3 2; STMF_PHASE_TIMING=1 timeout 300 python tools/diag_budget_run.py 4 25 2>&1 | tail -4; done 2>&1 | tee gpurun_out/prod_ab7.log; unset STMF_LIB
STMF_GRAPH=0 python tools/phaseB_capture.py 3 > /dev/null 2>&1 && \
STMF_GRAPH=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python tools/phaseB_capture.py 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
