#!/bin/bash
# Time each scan kernel row of kCfgs (CL_SCAN_CFG, scan_mamba1.cu) on a config.
CFG=${1:-C3}
for c in ${CFGS:-0 1 2 3}; do
  CL_SCAN_CFG=$c timeout 120 python tools/profile_stages.py --config $CFG --reps 12 --median 2>&1 | grep "cfg="
done
