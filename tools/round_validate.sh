set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo pytest=$? >> gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo smoke=$? >> gpurun_out/g_smoke.log
timeout 400 python bench.py > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_ref_c3.json 2>>gpurun_out/g_bench.err
for c in C1 C2; do timeout 300 python bench.py --config $c --no-producer > gpurun_out/g_bench_${c}.json 2>>gpurun_out/g_bench.err; done
timeout 500 python bench.py --config C4 --steps 20 --warmup 3 --no-producer --no-e2e > gpurun_out/g_bench_C4.json 2>>gpurun_out/g_bench.err
timeout 500 python bench.py --config C4 --chunk-policy guarded --steps 20 --warmup 3 --no-producer --no-e2e --no-cpu > gpurun_out/g_bench_C4g.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py sweep --config C2 > gpurun_out/g_sweep_c2.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py sweep --config C3 > gpurun_out/g_sweep_c3.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py mix > gpurun_out/g_mix.json 2>>gpurun_out/g_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-producer > gpurun_out/g_ncu.log 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:"rowpair_ws|hist_f32|minmax_f32" -c 3 -o gpurun_out/g_full python tools/profile_stages.py --config C3 --reps 1 > gpurun_out/g_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"rowpair_ws" -c 1 -o gpurun_out/g_full_c1 python tools/profile_stages.py --config C1 --reps 1 > gpurun_out/g_ncu2.log 2>&1
