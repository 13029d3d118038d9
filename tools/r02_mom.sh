set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_uq.py tests/test_gpu_benchsize.py tests/test_gpu_fullsize.py -q > gpurun_out/mo_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/mo_tests.txt
timeout 300 python bench.py --config mc > gpurun_out/mo_mc.json 2> gpurun_out/mo_mc.err
echo done
