#!/bin/bash
# A/B the L-parallel scan against the chained kernel on few-row shapes, and sweep its
# segment count (CL_LB_SEGS) and table row (lb:i).  Device time (graph replay, L2
# flushed), median of 15.   bash tools/lb_sweep.sh > gpurun_out/lb_sweep.txt
SHAPES=${SHAPES:-1x1536x2048,1x2048x4096,1x2048x8192,1x2048x32768,2x2048x4096,2x4096x2048,4x2048x4096,8x2048x2048}
python tools/cfg_ab.py $SHAPES chained,lb:0,lb:1,lb:2,lb:3,lb:4
for segs in ${SEGS:-6 8 12 16 20 24 32}; do
  echo "CL_LB_SEGS=$segs"
  CL_LB_SEGS=$segs python tools/cfg_ab.py 1x1536x2048,1x2048x4096 lb:0,lb:2,lb:3,lb:4
done
