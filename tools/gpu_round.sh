mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dropin or shard or prefill" > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log
