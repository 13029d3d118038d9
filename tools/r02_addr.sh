set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_benchsize.py tests/test_gpu_parity.py tests/test_gpu_parallel.py -x -q > gpurun_out/a_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/a_tests.txt
for rep in 1 2 3; do
  timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/a_new_$rep.json 2> gpurun_out/a_new_$rep.err
  FVB_LIB=$PWD/build/addrold/libfvb200.so timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/a_old_$rep.json 2> gpurun_out/a_old_$rep.err
done
echo done
