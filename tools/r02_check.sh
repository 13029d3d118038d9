# correctness pass on one B200: the GPU suite (+ new numerics / NCCL-skip tests), then the bench configs
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/c_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/c_tests.txt
timeout 300 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
timeout 300 python bench.py --config kh3d > gpurun_out/c_bench_kh3d.json 2> gpurun_out/c_bench_kh3d.err
timeout 300 python bench.py --config bqmc --steps 10 --no-cpu > gpurun_out/c_bench_bqmc.json 2> gpurun_out/c_bench_bqmc.err
echo done
