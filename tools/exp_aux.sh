timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in var_prev libstmf_b200; do echo $L; STMF_LIB=paper_2205_06619_b200/lib/$L.so timeout 400 python bench_fit.py --config 4 --seconds 15 | python3 -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['row_visits_per_s'], d['accepts'])"; done
