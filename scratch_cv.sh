for cv in default 0 50 100; do
  if [ $cv = default ]; then unset STMF_CARVEOUT; else export STMF_CARVEOUT=$cv; fi
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/cv.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('gpurun_out/cv.json')); print('$cv', round(d['ms_per_step'],1), round(d['roofline']['avg_launch_us'],1))"
done
