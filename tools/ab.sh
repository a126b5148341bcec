# A/B timing: each variant library in $LIBS ("default" = the in-tree build) on $CONFIG,
# then the GPU parity suite against the in-tree build.
set -e
for i in 1 2; do
for l in ${LIBS:-default}; do
  if [ "$l" = default ]; then unset CHUNKLAB_LIB; else export CHUNKLAB_LIB=$l; fi
  for c in ${CFGS:-default}; do
    if [ "$c" = default ]; then unset CL_SCAN_CFG; else export CL_SCAN_CFG=$c; fi
    echo -n "lib=$l "; python tools/profile_stages.py --config ${CONFIG:-C3} --reps 30 --median 2>&1 | grep cfg
  done
done
done
unset CHUNKLAB_LIB CL_SCAN_CFG
[ -n "$NOTEST" ] || timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
