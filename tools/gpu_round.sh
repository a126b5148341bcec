mkdir -p gpurun_out
./tools/micro/decide_lat > gpurun_out/r_decide_lat.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "entropy or hist or prefill or fullsize or robust or stress or lean or baseline or chunk or conv" > gpurun_out/r_tests.log 2>&1; echo rc=$? >> gpurun_out/r_tests.log
for i in 1 2; do timeout 300 python tools/profile_stages.py --config C3 --reps 30 --median 2>&1 | grep cfg; done > gpurun_out/r_c3.txt
