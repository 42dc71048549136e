#!/bin/bash
# Experiment (tools/): k_scen_fit occupancy (register cap via INTF_SCEN_FIT_MINB) vs duration
for B in 0 3 4; do
  INTF_NVCC_EXTRA="-DINTF_SCEN_FIT_MINB=$B" python -c "from paper_2512_18725_b200 import build; build.build(force=True)" 2>/dev/null
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_scen_fit|k_rls_g8|k_eval" python tools/c5_once.py 2>/dev/null | grep -E "k_scen_fit|k_rls|k_eval" | awk -F'","' -v b=$B '{print "minb " b ": " substr($5,1,40) " " $NF}'
done
