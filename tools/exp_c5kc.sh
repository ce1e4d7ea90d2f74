for K in 4 8 16; do echo "KC=$K"; STMF_C5_KC=$K timeout 600 python bench_c5.py --sizes 16384,65536 --ranks 16,64 --density 1.0 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], round(d['avg_ms'], 3), 'hbm', round(d['hbm']['frac'], 3), 'alu', round(d['alu']['frac'], 3), d['objective'])
"; done
