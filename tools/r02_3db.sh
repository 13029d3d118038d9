set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_parallel_dist.py tests/test_gpu_parallel.py -x -q > gpurun_out/u_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/u_tests.txt
for rep in 1 2; do
  timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/u_ks_$rep.json 2> gpurun_out/u_ks_$rep.err
  FVB_LIB=$PWD/build/r3late/libfvb200.so timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/u_late_$rep.json 2> gpurun_out/u_late_$rep.err
done
echo done
