mkdir -p gpurun_out
for i in 1 2; do for f in 256 64 1024 4096; do
  echo -n "F=$f "; CL_TOK_FLUSH_COST=$f timeout 300 python tools/profile_token.py --reps 10 2>&1 | tail -1
done; done > gpurun_out/v_ab.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "token" > gpurun_out/v_tests.log 2>&1; echo rc=$? >> gpurun_out/v_tests.log
