# bench configs (kh2d / mc / kh3d) + the process-per-rank tests on one B200
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parallel_dist.py tests/test_gpu_parallel.py tests/test_gpu_uq.py -x -q > gpurun_out/m_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/m_tests.txt
timeout 300 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
timeout 300 python bench.py --config mc > gpurun_out/m_bench_mc.json 2> gpurun_out/m_bench_mc.err
timeout 300 python bench.py --config kh3d > gpurun_out/m_bench_kh3d.json 2> gpurun_out/m_bench_kh3d.err
timeout 300 python bench.py --config bqmc --steps 10 --no-cpu > gpurun_out/m_bench_bqmc.json 2> gpurun_out/m_bench_bqmc.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err
echo done
