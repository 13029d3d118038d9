set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_benchsize.py tests/test_gpu_parity.py tests/test_gpu_parallel.py tests/test_gpu_fused_halo.py -x -q > gpurun_out/e_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/e_tests.txt
for rep in 1 2 3; do
  timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/e_noeq_$rep.json 2> gpurun_out/e_noeq_$rep.err
  FVB_LIB=$PWD/build/witheq/libfvb200.so timeout 200 python bench.py --no-cpu --e2e-reps 1 --steps 30 > gpurun_out/e_eq_$rep.json 2> gpurun_out/e_eq_$rep.err
done
echo done
