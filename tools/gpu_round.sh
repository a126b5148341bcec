mkdir -p gpurun_out
cp paper_2604_10597_b200/libchunklab_b200.so /tmp/new.so
for i in 1 2; do for l in /tmp/new.so build/variants/base.so; do
  export CHUNKLAB_LIB=$l; echo -n "$l "; timeout 300 python tools/profile_stages.py --config C3 --reps 30 --median 2>&1 | grep cfg
  echo -n "$l C1 "; timeout 300 python tools/profile_stages.py --config C1 --reps 30 --median 2>&1 | grep cfg
  echo -n "$l C2 "; timeout 300 python tools/profile_stages.py --config C2 --reps 30 --median 2>&1 | grep cfg
done; done > gpurun_out/ab_ab.txt
unset CHUNKLAB_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
