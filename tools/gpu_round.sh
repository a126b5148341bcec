mkdir -p gpurun_out
cp paper_2604_10597_b200/libchunklab_b200.so /tmp/new.so
for i in 1 2; do for l in /tmp/new.so build/variants/rev.so build/variants/ldcg.so build/variants/revldcg.so; do
  export CHUNKLAB_LIB=$l; echo -n "$l "; timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu --no-producer 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stage_breakdown_ms'].items()}, {k:round(v,4) for k,v in d['stage_ms'].items()}, d['clocks']['sm_mhz'])"
done; done > gpurun_out/ac_ab.txt
