#!/bin/bash
# host-side e2e parts at config 3 after the orientation / upload changes + the whole GPU suite
mkdir -p gpurun_out
python tools/diag_e2e_c3.py 2 2>&1 | tee gpurun_out/e2e_parts_c3.log
( time timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 ) 2>&1 | tail -10
