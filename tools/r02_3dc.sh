set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_parallel.py tests/test_gpu_parallel_dist.py -x -q > gpurun_out/v3_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/v3_tests.txt
for rep in 1 2; do timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/v3_kh3d_$rep.json 2> gpurun_out/v3_kh3d_$rep.err; done
FVB_BENCH_ARITH=exact timeout 300 python bench.py --config kh3d --no-cpu --cells 256 > gpurun_out/v3_exact3d.json 2> gpurun_out/v3_exact3d.err
echo done
