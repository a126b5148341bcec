mkdir -p gpurun_out
timeout 1000 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo pytest=$? >> gpurun_out/h_pytest.log
CHUNKLAB_LIB=build/variants/checked.so timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_lookback.py tests/test_gpu_stress.py tests/test_gpu_robustness.py tests/test_gpu_lean.py -x -q > gpurun_out/h_checked.log 2>&1; echo checked=$? >> gpurun_out/h_checked.log
for c in C1 C2; do timeout 300 python bench.py --config $c --no-producer --no-cpu > gpurun_out/h_bench_${c}.json 2>>gpurun_out/h_bench.err; done
timeout 400 python bench.py --no-cpu --no-producer > gpurun_out/h_bench_c3.json 2>>gpurun_out/h_bench.err
