#!/bin/bash
# One GPU round trip: -m gpu tests, a bench line of each arm, the phase-B launch list and
# one full ncu capture (host-driven loop: ncu cannot profile kernels inside conditional
# graphs), A/B variants of sweep 2.  Each profiled command first ran without ncu.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -6
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --ref-seconds 40 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
for v in "" "STMF_SPLIT=1" "STMF_UNROLL=4" "STMF_GROUP_MAJOR=1" "STMF_GRAPH=0"; do env $v python tools/s1_sweep.py 3 2; done 2>&1 | tee gpurun_out/ab.log
STMF_GRAPH=0 python tools/phaseB_capture.py 3 && \
STMF_GRAPH=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python tools/phaseB_capture.py 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
STMF_GRAPH=0 STMF_BATCH=256 python tools/phaseB_capture.py 3 && \
STMF_GRAPH=0 STMF_BATCH=256 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_phaseB -s 2 -c 1 -o gpurun_out/phaseB_c3 python tools/phaseB_capture.py 3 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
