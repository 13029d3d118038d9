set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_benchsize.py tests/test_gpu_parallel.py tests/test_gpu_parallel_dist.py -x -q > gpurun_out/v4_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/v4_tests.txt
for rep in 1 2; do timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/v4_kh3d_$rep.json 2> gpurun_out/v4_kh3d_$rep.err; done
timeout 600 python bench.py --config kh3d --no-cpu --cells 1024 --steps 5 --e2e-steps 2 > gpurun_out/v4_kh3d1024.json 2> gpurun_out/v4_kh3d1024.err
echo done
