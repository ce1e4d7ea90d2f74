#!/bin/bash
# round-end verification on one B200 (final kernels): the whole -m gpu suite, smoke, both bench arms,
# then the profiles: phase B at config 3 (ncu --set full, E = 256), the launch list of a config-3
# sweep-2 row window, k_product2 at config 4 (ncu --set full)
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 ) 2>&1 | tail -12
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_b200.json 2> gpurun_out/bench_b200.err; echo bench_rc=$?
tail -3 gpurun_out/bench_b200.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 --ref-seconds 40 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -3 gpurun_out/bench_ref.err
STMF_GRAPH=0 STMF_BATCH=256 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_phaseB -s 2 -c 1 -o gpurun_out/phaseB_c3_kpack python tools/phaseB_capture.py 3 > gpurun_out/ncu_phaseB_kpack.log 2>&1; echo ncu_phaseB=$?
STMF_GRAPH=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c3.csv python tools/phaseB_capture.py 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu_list=$?
STMF_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_product2 -s 6 -c 2 -o gpurun_out/prod_vec_c4 python tools/diag_budget_run.py 4 5 > gpurun_out/ncu_prod_vec.log 2>&1; echo ncu_prod=$?
