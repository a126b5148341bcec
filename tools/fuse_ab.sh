# A/B of the fused histogram -> decide launch (cl_histogram_decide_f32) against the
# separate decide kernel (CL_BENCH_SEPARATE_DECIDE=1), same library, C1/C2/C3 bench lines.
set -x
mkdir -p gpurun_out
for i in 1 2 3; do
for c in C1 C2 C3; do
  timeout 300 python bench.py --config $c --no-producer --no-e2e --no-cpu > gpurun_out/f_bench_${c}_fuse$i.json 2>>gpurun_out/f_bench.err
  CL_BENCH_SEPARATE_DECIDE=1 timeout 300 python bench.py --config $c --no-producer --no-e2e --no-cpu > gpurun_out/f_bench_${c}_sep$i.json 2>>gpurun_out/f_bench.err
done
done
