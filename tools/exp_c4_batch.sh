for B in "" "16,64,256" "32,128,512" "64,256,512" "128,512"; do
  echo "STMF_BATCH=$B"; STMF_BATCH=$B timeout 300 python tools/diag_phaseB_cfg.py 4 15 2>&1 | tail -1
done
