for E in "STMF_X=0" "STMF_UNROLL=4" "STMF_LONG=1024" "STMF_LONG=512" "STMF_UNROLL=4 STMF_LONG=1024"; do
  echo "$E"; env $E timeout 300 python tools/diag_phaseB_cfg.py 4 12 2>&1 | tail -1
done
for E in "STMF_X=0" "STMF_UNROLL=4" "STMF_LONG=1024" "STMF_LONG=512"; do
  echo "$E"; env $E timeout 300 python tools/diag_phaseB_cfg.py 3 6 2>&1 | tail -1
done
