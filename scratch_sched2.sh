for s in "1.5,4,2.0" "1.2,2,2.0" "1.0,2,1.5" "1.25,2,1.5" "0.9,1,1.5" "2.0,8,2.0" "1.0,1,2.0"; do
  STMF_SCHED=$s python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sch.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('gpurun_out/sch.json')); print('$s', round(d['ms_per_step'],1), d['evaluated_per_step'], d['roofline']['launches'])"
done
