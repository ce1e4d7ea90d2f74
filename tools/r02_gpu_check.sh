#!/bin/bash
# One GPU round trip: states, -m gpu tests, a bench line of each arm, the phase-B launch
# list and one full ncu capture (each profiled command first ran without ncu).
set -x
mkdir -p gpurun_out
python tools/make_states.py 2 > gpurun_out/states.log 2>&1; tail -12 gpurun_out/states.log
cp tests/golden/c*_state_s1.npz gpurun_out/
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -6
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 20 > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --ref-seconds 40 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
python tools/phaseB_capture.py 3 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/phaseB_capture.py 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_phaseB -s 3 -c 1 -o gpurun_out/phaseB_c3 python tools/phaseB_capture.py 3 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
