mkdir -p gpurun_out
for v in default poly1; do
  if [ $v = default ]; then unset CHUNKLAB_LIB; else export CHUNKLAB_LIB=build/variants/$v.so; fi
  timeout 300 python tools/profile_stages.py --config C3 --reps 1 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:"rowpair_ws" -c 1 -o gpurun_out/k_$v python tools/profile_stages.py --config C3 --reps 1 > gpurun_out/k_ncu_$v.log 2>&1
done
