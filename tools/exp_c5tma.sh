timeout 300 python -m pytest tests/test_gpu_maxplus.py -q 2>&1 | tail -2
for T in 0 1; do echo "TMA=$T"; STMF_C5_TMA=$T timeout 600 python bench_c5.py --sizes 16384,65536 --ranks 4,16,64 --density 1.0,0.1 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], round(d['avg_ms'], 3), 'hbm', round(d['hbm']['frac'], 3), 'alu', round(d['alu']['frac'], 3), d['objective'])
"; done
