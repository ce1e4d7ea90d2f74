for S in "" "0.9,1,2.0"; do echo "SCHED=$S"; STMF_SCHED=$S timeout 400 python tools/diag_sweep_times.py 3 3 | grep "^sweep" | cut -c1-60; done
