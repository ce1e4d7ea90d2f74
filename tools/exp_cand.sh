timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 100 python tools/diag_sweep_times.py 2 8 | grep "^sweep" | tail -4 | cut -c1-30
timeout 300 python bench_fit.py --config 3 --sweeps 2 | cut -c1-400
