#!/bin/bash
# A/B of the L-parallel kernel's knobs: aggregate-pass software pipeline (CL_LB_PIPE1) and
# the split's cost model (CL_LB_PHI: relative cost of the aggregate pass).  Device time.
SHAPES=${SHAPES:-1x1536x2048,1x2048x4096,1x2048x8192,1x2048x32768,2x2048x4096}
for pipe in 0 1; do for phi in 0 0.3 0.6; do
  echo "PIPE1=$pipe PHI=$phi"
  CL_LB_PIPE1=$pipe CL_LB_PHI=$phi python tools/cfg_ab.py $SHAPES lb:0,lb:3
done; done
