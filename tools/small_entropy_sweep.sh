#!/bin/bash
# C1/C2 step time vs the small-input launch shapes of the entropy stages:
# CL_MM_CTAS_PER_SM (min/max grid) x CL_HIST_MIN_CHUNKS (register-fed histogram grid).
for c in ${CONFIGS:-C1 C2}; do for mm in 4 8; do for hc in 1 2 4 8; do
  CL_MM_CTAS_PER_SM=$mm CL_HIST_MIN_CHUNKS=$hc python bench.py --config $c --steps 60 --warmup 5 \
    --no-e2e --no-cpu --no-producer 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c mm=$mm hc=$hc step', round(d['ms_per_step'],5), 'entropy', round(d['stage_ms']['entropy'],5), 'scan', round(d['stage_ms']['scan'],5), d['stage_breakdown_ms'])"
done; done; done
