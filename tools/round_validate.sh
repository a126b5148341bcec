# The round's evidence pack on one GPU box (outputs under gpurun_out/g_*; copy to profiles/):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/round_validate.sh'
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo pytest=$? >> gpurun_out/g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo smoke=$? >> gpurun_out/g_smoke.log
timeout 600 python bench.py > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_ref_c3.json 2>>gpurun_out/g_bench.err
for c in C1 C2; do timeout 300 python bench.py --config $c --no-producer > gpurun_out/g_bench_${c}.json 2>>gpurun_out/g_bench.err; done
timeout 500 python bench.py --config C4 --steps 20 --warmup 3 --no-producer --no-e2e > gpurun_out/g_bench_C4.json 2>>gpurun_out/g_bench.err
timeout 500 python bench.py --config C4 --chunk-policy guarded --steps 20 --warmup 3 --no-producer --no-e2e --no-cpu > gpurun_out/g_bench_C4g.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py sweep --config C2 > gpurun_out/g_sweep_c2.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py sweep --config C3 > gpurun_out/g_sweep_c3.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/chunk_sweep.py mix > gpurun_out/g_mix.json 2>>gpurun_out/g_bench.err
timeout 300 python tools/profile_token.py --reps 10 > gpurun_out/g_token.txt 2>>gpurun_out/g_bench.err
for c in C1 C3; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-producer > gpurun_out/g_ncu_$c.log 2>&1
done
for c in C1 C2 C3; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"rowpair_ws|lookback_ws" -c 1 --csv --log-file gpurun_out/traffic_$c.csv python tools/scan_traffic.py --run $c > gpurun_out/g_tr_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rowpair_ws|hist_f32_reg|minmax_f32" -c 3 -o gpurun_out/g_full python tools/profile_stages.py --config C3 --reps 1 > gpurun_out/g_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"lookback_ws" -c 1 -o gpurun_out/g_full_c1 python tools/profile_stages.py --config C1 --reps 1 > gpurun_out/g_ncu2.log 2>&1
