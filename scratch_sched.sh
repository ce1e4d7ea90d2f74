for s in "1.25,2,2.0" "1.0,1,1.5" "1.1,1,2.0" "0.8,1,1.5" "1.5,4,2.0"; do
  echo "S=$s"
  STMF_SCHED=$s python scratch_time.py 2 6 2>&1 | grep "sweep 6" | cut -c1-30
  STMF_SCHED=$s timeout 300 python bench_fit.py --config 3 --seconds 12 --warm-sweeps 1 2>&1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['row_visits_per_s'],1), round(d['evaluated']/d['attempts'],2))"
done
