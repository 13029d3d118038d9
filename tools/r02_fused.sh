set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_halo.py tests/test_gpu_parallel_dist.py tests/test_gpu_parallel.py -q > gpurun_out/fh_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/fh_tests.txt
timeout 300 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/fh_bench.json 2> gpurun_out/fh_bench.err
timeout 300 python bench.py --config kh3d --no-cpu > gpurun_out/fh_kh3d.json 2> gpurun_out/fh_kh3d.err
echo done
