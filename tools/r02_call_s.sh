#!/bin/bash
# first-batch scale for rows WITH depth history (real fits; the bench window has none): config 3 sweeps 1-5
mkdir -p gpurun_out
for s in 0.9,1,1.15 0.6,1,1.15 0.4,1,1.15 0.25,1,1.15 0.0,16,1.15; do
  echo "== SCHED=$s"
  STMF_SCHED=$s timeout 600 python tools/long_fit.py 3 5 600 gpurun_out/c3_sched_tmp.jsonl 2>&1 | python -c "
import sys, json
t = 0
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if 'sweep' in d:
        t += d['seconds']; print(d['sweep'], round(d['seconds'], 2), d['attempts'], d['evaluated'], d['error'])
print('total', round(t, 2))
"
done 2>&1 | tee gpurun_out/ab12_hist_scale.log
rm -f gpurun_out/c3_sched_tmp*
