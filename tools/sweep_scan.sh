#!/bin/bash
# Time each scan geometry (CL_SCAN_CFG) on a config; prints stage times per cfg.
CFG=${1:-C3}
for c in ${CFGS:-0 1 2 3 4 5 6 7 8 9 10 11 12 13 14}; do
  echo "cfg $c: $(CL_SCAN_CFG=$c timeout 120 python tools/profile_stages.py --config $CFG --reps 4 2>&1 | head -1)"
done
