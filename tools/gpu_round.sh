mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
timeout 500 python bench.py --config C4 --chunk-policy guarded --steps 20 --warmup 3 --no-producer --no-e2e --no-cpu > gpurun_out/w_bench_C4g.json 2>gpurun_out/w_bench.err
