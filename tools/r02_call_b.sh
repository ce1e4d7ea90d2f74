#!/bin/bash
# lane-coded config-5 kernel (tests + timings), the FitRun protocol test, an ncu capture of
# k_product2 at config 4, then the config-3 long fit from the state after sweep 37
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxplus.py tests/test_gpu_fitrun.py -x -q 2>&1 | tail -8
STMF_C5_VERBOSE=1 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes,dense 2>&1 | tee gpurun_out/c5_lanes2_a.jsonl
for st in 1 2 3; do echo "stages=$st"; STMF_C5_VERBOSE=1 STMF_C5_STAGES=$st python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes 2>&1 | python -c "import sys,json; [print(l.strip() if not l.startswith('{') else (json.loads(l)['avg_ms'], json.loads(l)['hbm']['frac'])) for l in sys.stdin]"; done 2>&1 | tee gpurun_out/c5_lanes2_sweep.log
python bench_c5.py --sizes 4096,16384,65536 --ranks 4,16 --density 0.1,0.5 --layouts lanes 2>&1 | tee gpurun_out/c5_lanes2_b.jsonl
python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes --reps 2 > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_maxplus_err_lanes -s 1 -c 1 -o gpurun_out/c5_lanes2 python bench_c5.py --sizes 65536 --ranks 4 --density 0.1 --layouts lanes --reps 2 > gpurun_out/ncu_lanes2.log 2>&1; echo ncu_lanes=$?
timeout 300 python tools/diag_budget_run.py 4 5 > /dev/null 2>&1 && \
STMF_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_product2 -s 6 -c 2 -o gpurun_out/prod2_c4 python tools/diag_budget_run.py 4 5 > gpurun_out/ncu_prod2.log 2>&1; echo ncu_prod=$?
timeout 2250 python tools/long_fit.py 3 200 2000 gpurun_out/c3_long_part3.jsonl profiles/states/c3_after_sweep37.npz 38 2>&1 | tail -16
