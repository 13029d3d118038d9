set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parallel_dist.py tests/test_gpu_reference_suite.py tests/test_gpu_bench_contract.py -q > gpurun_out/f_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.txt
bash tools/r02_ncu_all.sh
